"""CG iterations of the AMG-PCG frame vs pcg_tol on a scaled c5 (QN_AMG_ZF=0/1 A/B)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import paper_1604_07378_b200 as Q
from paper_1604_07378_b200 import scenes
from test_gpu_parity import build

for grid in ((20, 6, 6), (60, 15, 15)):
    for tol in (1e-10, 1e-11, 1e-12, 1e-13):
        sc = scenes.c5(grid=grid, frames=1)
        system = build(sc, solver="amg", pcg_tol=tol)
        run = Q.ResidentRun(system, Q.SimState(q_l=np.array(sc.q_l), q_prev=np.array(sc.q_prev)),
                            Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
        try:
            run.step()
            print(grid, "tol", tol, "cg iterations", run.last_cg_iterations, flush=True)
        except Exception as ex:
            print(grid, "tol", tol, "FAILED", str(ex)[:90], "cg", run.last_cg_iterations, flush=True)
