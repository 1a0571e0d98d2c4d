"""Tiny instances of every device path, for compute-sanitizer (one tool per run):

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

frame graph (direct solve, dense top, batch), host-driven loop, PCG / AMG,
colliders, ARAP, fibres, springs, Chebyshev, scaled-identity L-BFGS, the
slab frame (two emulated slabs with the coarse level) and the seams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1604_07378_b200 as Q  # noqa: E402
from paper_1604_07378_b200 import dynamics as D, scenes, slab  # noqa: E402
from paper_1604_07378_b200.materials import PDMaterial, from_spec  # noqa: E402


def frames(system, sc, cfg, n=2):
    st = Q.SimState(q_l=np.array(sc.q_l), q_prev=np.array(sc.q_prev))
    for _ in range(n):
        st, rec = Q.simulate_frame(system, st, cfg)
    return st


def build(sc, **kw):
    return Q.build_system(Q.TetMesh(sc.verts, sc.tets, sc.density), kw.pop("mat", None) or from_spec(sc.material),
                          h=sc.h, gravity=sc.gravity, fixed=sc.fixed, **kw)


def main():
    sc = scenes.c1(grid=(6, 2, 2), iterations=6)
    lb = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    frames(build(sc), sc, lb)
    s = build(sc)
    s.set_graph_mode(False)
    frames(s, sc, lb)
    frames(build(sc, solver="pcg"), sc, lb)
    frames(build(sc, solver="amg"), sc, lb)
    frames(build(sc, colliders=[D.HalfSpace((0, 0, -0.02), (0, 0, 1)), D.SphereCollider((0.3, 0.1, -0.2), 0.2),
                                D.TorusCollider((0.2, 0.1, -0.1), 0.1, 0.05)]), sc, lb)
    frames(build(sc, mat=PDMaterial("arap", 1e5)), sc, lb)
    frames(build(sc, aniso=[(e, (1, 0, 0), 1e5) for e in range(sc.tets.shape[0])]), sc, lb)
    frames(build(sc), sc, Q.SolverConfig(kind="chebyshev", iterations=sc.iterations, S=2))
    frames(build(sc), sc, Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, lbfgs_init="scaled_identity"))
    c2 = scenes.c2(grid=(12, 4, 4), iterations=4)
    frames(build(c2), c2, Q.SolverConfig(kind="lbfgs", iterations=c2.iterations, m=c2.m))
    b = Q.build_batch_system(Q.TetMesh(sc.verts, sc.tets, sc.density), [from_spec(sc.material)] * 3, h=sc.h,
                             gravity=sc.gravity, fixed=sc.fixed)
    st = Q.SimState(q_l=np.stack([sc.q_l] * 3), q_prev=np.stack([sc.q_prev] * 3))
    Q.simulate_frame(b, st, lb)
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cloth = Q.load_obj_springs(os.path.join(here, "tests", "golden", "ref_fixtures", "cloth20.obj"), 0.2)
    cs = Q.build_system(cloth, PDMaterial("mass_spring", 200.0), fixed=[0, 19])
    Q.simulate_frame(cs, Q.SimState(q_l=cloth.vertices.copy(), q_prev=cloth.vertices.copy()), lb)
    s5 = scenes.c5(grid=(8, 2, 2), frames=1, iterations=3)
    ranks = slab.scene_slabs(s5, 2)
    comm = slab.EmulatedComm(ranks)
    slab.setup_coarse(comm, s5.grid, (4, 2, 2))
    slab.SlabRun(comm, Q.SolverConfig(kind="lbfgs", iterations=3), s5.h, slab.scene_grad_tol(s5)).step()
    s1 = build(sc)
    x = sc.q_l + 1e-3
    Q.svd_rv_batch(np.random.default_rng(0).standard_normal((50, 3, 3)))
    st = Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev)
    st.y = Q.inertia_target(st, s1)
    Q.objective(s1, st, x)
    Q.gradient(s1, st, x)
    print("sanitize cases done")


if __name__ == "__main__":
    main()
