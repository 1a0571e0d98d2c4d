"""Per-tet kernel on a deformed state of a workload, for the fp64 flop count
(ncu sass counters) per material:

    ncu --metrics smsp__sass_thread_inst_executed_op_d{fma,mul,add}_pred_on.sum,gpu__time_duration.sum \
        -k regex:k_tet_plain python tools/tet_flops.py c3 [nx ny nz]

Runs `frames` frames (graph mode, kernels k_tet) so the state is deformed, then
three stand-alone k_tet_plain launches at the resident positions (the launches
ncu's -k filter keeps)."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402

import paper_1604_07378_b200 as Q  # noqa: E402
from paper_1604_07378_b200 import scenes  # noqa: E402

sys.argv += [] if len(sys.argv) > 1 else ["c3"]
name = sys.argv[1]
kw = {"grid": tuple(int(a) for a in sys.argv[2:5])} if len(sys.argv) >= 5 else {}
sc = scenes.CONFIGS[name](**kw)
import bench  # noqa: E402

system = bench.build_system(sc)
cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
run = Q.ResidentRun(system, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev), cfg)
for _ in range(3):
    run.step()
ms = system.time_kernel("tet", reps=2)
print(f"{name} tets {sc.tets.shape[0]} x {max(1, sc.batch)} instances: k_tet_plain {ms * 1e3:.1f} us")
