"""Live per-pass timeline of one frame inside the CUDA graph (diagnostics):
for every body pass, when k_grad, k_eta, k_vec and k_tet start (block 0
entry) and when their finalising block ends; the solve is the interval
between k_grad's end and k_eta's start.

    python tools/frame_timeline.py [c2] [frames]
"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1604_07378_b200 as Q  # noqa: E402
from paper_1604_07378_b200 import _lib  # noqa: E402
from paper_1604_07378_b200.solvers import ResidentRun, SolverConfig  # noqa: E402

PASSES, KERNELS = 512, 7


def main(cfg="c2", frames="3"):
    import bench
    sc = bench.build_scene(cfg, 0, 1)
    system = bench.build_system(sc)
    lib = _lib.load()
    run = ResidentRun(system, Q.SimState(sc.q_l, sc.q_prev), SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
    for _ in range(2):
        run.step()
    _lib.check(lib.qn_system_set_timeline(system._h, 1))
    buf = np.zeros(PASSES * KERNELS * 2, dtype=np.uint64)
    for _ in range(int(frames)):
        run.step()
    _lib.check(lib.qn_system_timeline(system._h, _lib.ptr(buf), C.c_int64(buf.size)))
    t = buf.reshape(PASSES, KERNELS, 2).astype(np.int64)
    npass = int((t[:, 3, 1] > 0).sum())
    t0 = t[0, 0, 0] if t[0, 0, 0] else t[0, 3, 0]
    rows = []
    for p in range(npass):
        g0, g1 = t[p, 0]
        e0, e1 = t[p, 1]
        v0 = t[p, 2, 0]
        k0, k1 = t[p, 3]
        rows.append(((g1 - g0) if g0 and g1 else 0, (e0 - g1) if g1 and e0 else 0, (v0 - e0) if e0 and v0 else 0,
                     (k0 - v0) if v0 else 0, k1 - k0, (t[p + 1, 0, 0] - k1) if p + 1 < npass else 0))
    r = np.array(rows, dtype=np.float64) / 1000.0
    sv = [(t[p, 4, 0] - t[p, 0, 1], t[p, 4, 1] - t[p, 4, 0], t[p, 5, 0] - t[p, 4, 1], t[p, 5, 1] - t[p, 5, 0],
           t[p, 1, 0] - t[p, 5, 1]) for p in range(npass) if t[p, 4, 0] and t[p, 5, 1] and t[p, 0, 1] and t[p, 1, 0]]
    full = r[:, 1] > 0  # passes with a direction (grad + solve + eta)
    names = ["grad", "grad_end->eta (solve)", "eta (entry->vec entry)", "vec", "tet", "tet_end->next grad"]
    print(f"{cfg}: {npass} passes in the last frame, {full.sum()} with a solve; "
          f"frame span {(t[npass - 1, 3, 1] - t0) / 1000.0:.1f} us")
    for j, n in enumerate(names):
        sel = r[full, j] if j < 3 else r[:, j]
        print(f"  {n:24s} mean {sel.mean():7.2f} us  min {sel.min():7.2f}  max {sel.max():7.2f}")
    if sv:
        a = np.array(sv, dtype=np.float64) / 1000.0
        for j, n in enumerate(["grad end -> fwd entry", "forward", "fwd end -> bwd entry", "backward",
                               "bwd end -> eta entry"]):
            print(f"    {n:22s} mean {a[:, j].mean():7.2f} us")
        tp = [(t[p, 6, 0] - t[p, 4, 1], t[p, 6, 1] - t[p, 6, 0], t[p, 5, 0] - t[p, 6, 1]) for p in range(npass)
              if t[p, 6, 0] and t[p, 6, 1] and t[p, 4, 1] and t[p, 5, 0]]
        if tp:
            a = np.array(tp, dtype=np.float64) / 1000.0
            for j, n in enumerate(["fwd end -> top entry", "top", "top end -> bwd entry"]):
                print(f"      {n:22s} mean {a[:, j].mean():7.2f} us")


if __name__ == "__main__":
    main(*sys.argv[1:])
