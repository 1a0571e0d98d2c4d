"""One stand-alone AMG V-cycle of configs[4] after a frame (for ncu):

    ncu --set full -k regex:k_amg -c 22 python tools/vcycle_profile.py
"""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1604_07378_b200 as Q  # noqa: E402
import bench  # noqa: E402

sc = bench.build_scene("c5", 0, 1)
system = bench.build_system(sc)
run = Q.ResidentRun(system, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev),
                    Q.SolverConfig(kind="lbfgs", iterations=2, m=sc.m))
run.step()
ms = system.time_kernel("vcycle", reps=1)
print(f"vcycle {ms:.3f} ms", system.amg_info())
