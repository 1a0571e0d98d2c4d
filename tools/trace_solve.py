"""Timeline of one traced supernodal solve (diagnostics): per group of tickets,
when tasks take their ticket, finish staging, see their dependencies ready,
and how long the gather / compute / publish phases take (SM clock64).

    python tools/trace_solve.py [c2] [plain|graph]

plain: a stand-alone solve through the factor API (PlainIO);
graph: the last solve of a real frame inside the CUDA graph (SolverIO).
"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1604_07378_b200 as Q  # noqa: E402
from paper_1604_07378_b200 import _lib  # noqa: E402
from paper_1604_07378_b200.solvers import ResidentRun, SolverConfig  # noqa: E402

SLOTS = 9
GHZ = 1.965  # SM clock under load (bench clocks line)


def report(name, st7, t):
    st7 = st7[:, :7]
    st = np.zeros((st7.shape[0], 6), dtype=np.int64)
    st[:, 0], st[:, 1], st[:, 2] = st7[:, 0], st7[:, 1], st7[:, 2]
    for j in range(3):  # phases after 'ready' from the SM cycle counter
        st[:, 3 + j] = st7[:, 2] + ((st7[:, 4 + j] - st7[:, 3]) / GHZ).astype(np.int64)
    ok = st[:, 0] > 0
    st, t = st[ok], t[ok]
    s = (st - st[:, 0].min()) / 1000.0
    print(f"--- {name}: {len(t)} tasks, span {s[:, 5].max():.1f} us | mean staging {np.mean(s[:, 1] - s[:, 0]):.2f} "
          f"wait {np.mean(s[:, 2] - s[:, 1]):.2f} gather {np.mean(s[:, 3] - s[:, 2]):.2f} "
          f"compute {np.mean(s[:, 4] - s[:, 3]):.2f} publish {np.mean(s[:, 5] - s[:, 4]):.2f} us")
    for idx in np.array_split(np.arange(len(t)), 12):
        print(f"  tickets {idx[0]:5d}-{idx[-1]:5d}: ticket {s[idx, 0].min():7.1f}..{s[idx, 0].max():7.1f} "
              f"ready {np.median(s[idx, 2]):7.1f} end {s[idx, 5].max():7.1f} | staging "
              f"{np.mean(s[idx, 1] - s[idx, 0]):5.2f} wait {np.mean(s[idx, 2] - s[idx, 1]):5.2f} gather "
              f"{np.mean(s[idx, 3] - s[idx, 2]):5.2f} compute {np.mean(s[idx, 4] - s[idx, 3]):5.2f} publish "
              f"{np.mean(s[idx, 5] - s[idx, 4]):5.2f}")


def main(cfg="c2", mode="plain"):
    import bench
    sc = bench.build_scene(cfg, 0, 1)
    system = bench.build_system(sc)
    lib = _lib.load()
    f = system.sysfact
    nf, nb = C.c_int64(), C.c_int64()
    _lib.check(lib.qn_factor_task_counts(f._h, C.byref(nf), C.byref(nb)))
    nf, nb = nf.value, nb.value
    stamps = np.zeros(SLOTS * (nf + nb), dtype=np.uint64)
    tasks = np.zeros(4 * (nf + nb), dtype=np.int32)
    if mode == "graph":
        run = ResidentRun(system, Q.SimState(sc.q_l, sc.q_prev), SolverConfig(iterations=sc.iterations, m=sc.m))
        run.step()
        _lib.check(lib.qn_system_set_timeline(system._h, 1))
        run.step()
        _lib.check(lib.qn_system_solve_trace(system._h, _lib.ptr(stamps), _lib.ptr(tasks)))
        _lib.check(lib.qn_system_set_timeline(system._h, 0))
    else:
        B = np.random.default_rng(0).standard_normal((f.n, 3))
        for _ in range(5):
            f.solve(B)
        for _ in range(3):
            _lib.check(lib.qn_factor_trace_solve(f._h, _lib.ptr(stamps), _lib.ptr(tasks)))
    st = stamps.reshape(-1, SLOTS).astype(np.int64)
    tk = tasks.reshape(-1, 4)
    print(cfg, mode, f.info())
    report("forward", st[:nf], tk[:nf])
    report("backward", st[nf:nf + nb], tk[nf:nf + nb])
    import os
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez(f"gpurun_out/trace_{cfg}_{mode}.npz", st=st, tk=tk, nf=nf, nb=nb)


if __name__ == "__main__":
    main(*sys.argv[1:])
