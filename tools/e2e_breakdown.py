"""Host-side breakdown of one simulate_frame call (diagnostics): state upload,
frame, download and record conversion, for a config (default c4).

    python tools/e2e_breakdown.py [c4]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1604_07378_b200 as Q  # noqa: E402
from paper_1604_07378_b200 import _lib  # noqa: E402
from paper_1604_07378_b200.solvers import _RecordBuffers  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    sc = bench.build_scene(name, 0, 1)
    system = bench.build_system(sc)
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    shape = np.asarray(sc.q_l).shape
    pin = [torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)]
    pin[0][...] = sc.q_l
    pin[1][...] = sc.q_prev
    lib = _lib.load()
    c = cfg.to_c()
    for rep in range(4):
        t = [time.perf_counter()]
        _lib.check(lib.qn_state_set(system._h, _lib.ptr(pin[0]), _lib.ptr(pin[1]), _lib.QN_MEM_HOST, None))
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        rb = _RecordBuffers(system.n_inst, cfg.iterations)
        _lib.check(lib.qn_frame_step(system._h, C.byref(c), None, C.byref(rb.c), _lib.QN_MEM_HOST, 1, None))
        t.append(time.perf_counter())
        _lib.check(lib.qn_state_get(system._h, _lib.ptr(pin[2]), None, _lib.ptr(pin[3]), _lib.QN_MEM_HOST, None))
        t.append(time.perf_counter())
        recs = rb.records()
        t.append(time.perf_counter())
        st = Q.SimState(q_l=pin[0], q_prev=pin[1])
        t0 = time.perf_counter()
        Q.simulate_frame(system, st, cfg, out=Q.SimState(q_l=pin[2], q_prev=pin[0], y=pin[3]))
        t1 = time.perf_counter()
        dt = np.diff(t) * 1e3
        print(f"upload {dt[0]:.2f} ms | frame+records {dt[1]:.2f} | download {dt[2]:.2f} | records->python {dt[3]:.2f}"
              f" | device frame {system_ms(system):.2f} | whole simulate_frame {1e3 * (t1 - t0):.2f} ms")


def system_ms(system):
    v = C.c_double(0.0)
    _lib.check(_lib.load().qn_system_last_frame_ms(system._h, C.byref(v)))
    return v.value


if __name__ == "__main__":
    main()
