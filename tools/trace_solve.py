"""Timeline of one traced supernodal solve (diagnostics): per tree level, when
tasks start, when their dependencies are ready and when they finish.

    python tools/trace_solve.py [c2]
"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1604_07378_b200 as Q  # noqa: E402
from paper_1604_07378_b200 import _lib, scenes  # noqa: E402
from paper_1604_07378_b200.materials import from_spec  # noqa: E402


def main(cfg="c2"):
    sc = scenes.CONFIGS[cfg]()
    system = Q.build_system(Q.TetMesh(sc.verts, sc.tets, sc.density), from_spec(sc.material), h=sc.h,
                            gravity=sc.gravity, fixed=sc.fixed)
    f = system.sysfact
    B = np.random.default_rng(0).standard_normal((f.n, 3))
    for _ in range(5):
        f.solve(B)
    nf, nb = C.c_int64(), C.c_int64()
    lib = _lib.load()
    _lib.check(lib.qn_factor_task_counts(f._h, C.byref(nf), C.byref(nb)))
    nf, nb = nf.value, nb.value
    stamps = np.zeros(6 * (nf + nb), dtype=np.uint64)
    tasks = np.zeros(4 * (nf + nb), dtype=np.int32)
    for _ in range(3):
        _lib.check(lib.qn_factor_trace_solve(f._h, _lib.ptr(stamps), _lib.ptr(tasks)))
    st6 = stamps.reshape(-1, 6).astype(np.int64)
    ghz = 1.965  # SM clock under load (bench clocks line)
    st = np.zeros((st6.shape[0], 5), dtype=np.int64)
    st[:, 0], st[:, 1] = st6[:, 0], st6[:, 1]
    for j in range(3):  # phases after 'ready' from the SM cycle counter
        st[:, 2 + j] = st6[:, 1] + ((st6[:, 3 + j] - st6[:, 2]) / ghz).astype(np.int64)
    tk = tasks.reshape(-1, 4)
    info = f.info()
    print(cfg, info)
    for name, sl in (("forward", slice(0, nf)), ("backward", slice(nf, nf + nb))):
        s = st[sl]
        t = tk[sl]
        t0 = s[:, 0].min()
        s = (s - t0) / 1000.0
        sup = t[:, 0]
        # level of each supernode = its position in the ticket order groups (height / depth)
        order_levels = {}
        lvl = np.zeros(len(t), dtype=int)
        # recompute levels from ticket order: consecutive supernodes share a level when monotone
        par = None
        print(f"--- {name}: {len(t)} tasks, span {s[:, 4].max():.1f} us, "
              f"mean wait {np.mean(s[:, 1] - s[:, 0]):.2f} us, mean work {np.mean(s[:, 4] - s[:, 1]):.2f} us "
              f"(gather {np.mean(s[:, 2] - s[:, 1]):.2f} compute {np.mean(s[:, 3] - s[:, 2]):.2f} "
              f"publish {np.mean(s[:, 4] - s[:, 3]):.2f})")
        # bucket by completion-time deciles of the task list order
        q = np.array_split(np.arange(len(t)), 12)
        for i, idx in enumerate(q):
            print(f"  tickets {idx[0]:5d}-{idx[-1]:5d}: start {s[idx,0].min():7.1f}..{s[idx,0].max():7.1f} "
                  f"ready {np.median(s[idx,1]):7.1f} end {s[idx,4].max():7.1f}  "
                  f"wait {np.mean(s[idx,1]-s[idx,0]):5.2f} gather {np.mean(s[idx,2]-s[idx,1]):5.2f} "
                  f"compute {np.mean(s[idx,3]-s[idx,2]):5.2f} publish {np.mean(s[idx,4]-s[idx,3]):5.2f} us")


if __name__ == "__main__":
    main(*sys.argv[1:])
