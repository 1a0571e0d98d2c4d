"""configs[4] parity vs PCG tolerance: the single-system AMG-PCG frame (and
the emulated 2/4-slab frame) against a reference frame that is exact to ~1e-13
(the CG oracle, or a committed golden), for pcg_tol = 1e-10 .. 1e-13.

    python tools/c5_tol_sweep.py [nx ny nz] [--golden tests/golden/frames_c5_200x50x50.npz]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1604_07378_b200 as Q  # noqa: E402
from paper_1604_07378_b200 import scenes, slab  # noqa: E402
from paper_1604_07378_b200.materials import from_spec  # noqa: E402


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("grid", type=int, nargs="*", default=[40, 10, 10])
    ap.add_argument("--golden", default=None)
    ap.add_argument("--frames", type=int, default=2)
    ap.add_argument("--slabs", type=int, nargs="*", default=[])
    ap.add_argument("--tols", type=float, nargs="*", default=[1e-10, 1e-11, 1e-12, 1e-13])
    a = ap.parse_args()
    if a.golden:
        d = np.load(a.golden)
        grid = tuple(int(v) for v in d["grid"])
        frames = min(a.frames, int(d["frames"]))
        ref = [(d[f"x_{f}"], list(d[f"g_{f}"]), list(d[f"trials_{f}"])) for f in range(frames)]
        ids = d["ids"]
    else:
        import oracle.qnsim_oracle as O
        from tests.helpers import oracle_material
        grid, frames = tuple(a.grid), a.frames
        sc = scenes.c5(grid=grid)
        osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                       factor="sparse")
        ql, qp = sc.q_l.copy(), sc.q_prev.copy()
        ref, ids = [], np.arange(sc.verts.shape[0])
        for _ in range(frames):
            x, _, r = O.simulate_frame(osys, ql, qp, iterations=sc.iterations, m=sc.m)
            qp, ql = ql, x
            ref.append((x, r.g, r.ls_trials))
    sc = scenes.c5(grid=grid)
    for tol in a.tols:
        t = time.time()
        system = Q.build_system(Q.TetMesh(sc.verts, sc.tets, sc.density), from_spec(sc.material), h=sc.h,
                                gravity=sc.gravity, fixed=sc.fixed, solver="amg", pcg_tol=tol)
        bt = time.time() - t
        run = Q.ResidentRun(system, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev),
                            Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
        for f in range(frames):
            rec = run.step(record=True)[0]
            x = run.state().q_l
            xr, gr, tr = ref[f]
            print(f"grid {grid} single AMG tol {tol:.0e} frame {f}: dx {rel(x[ids], xr):.2e} dg {rel(rec.g, gr):.2e} "
                  f"trials_equal {list(rec.ls_trials) == list(tr)} cg {run.last_cg_iterations} "
                  f"frame_ms {run.last_ms:.1f} build_s {bt:.1f}", flush=True)
        del run, system
        for world in a.slabs:
            ranks = slab.scene_slabs(sc, world, solver="amg", pcg_tol=tol)
            comm = slab.EmulatedComm(ranks)
            slab.setup_coarse(comm, sc.grid, (8, 2, 2))
            srun = slab.SlabRun(comm, Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m), sc.h,
                                slab.scene_grad_tol(sc))
            for f in range(frames):
                rec = srun.step()
                x = slab.gather_positions(ranks)
                xr, gr, tr = ref[f]
                print(f"grid {grid} slabs {world} tol {tol:.0e} frame {f}: dx {rel(x[ids], xr):.2e} "
                      f"dg {rel(rec.g, gr):.2e} trials_equal {list(rec.ls_trials) == list(tr)}", flush=True)
            del srun, comm, ranks


if __name__ == "__main__":
    main()
