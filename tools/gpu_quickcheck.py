"""Ad-hoc GPU diagnostics: SVD, factor solve, objective/gradient, frames vs the oracle."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle.qnsim_oracle as O
import paper_1604_07378_b200 as Q
from paper_1604_07378_b200 import scenes, materials as M


def omat(spec):
    f = {"zero": lambda s: O.Zero(), "poly": lambda s: O.Poly(s[1]), "log": lambda s: O.Log(s[1], s[2]),
         "hermite": lambda s: O.Hermite(s[1])}
    return O.VLMaterial(*[f[x[0]](x) for x in spec])


def main(name="c1", frames=3, graph=True):
    rng = np.random.default_rng(5)
    # --- SVD
    F = rng.standard_normal((20000, 3, 3))
    F[:100] = np.eye(3) + 1e-9 * rng.standard_normal((100, 3, 3))
    F[100:200] *= np.array([1, 1, -1.0])[None, :, None]
    F[200:300, :, 2] = 0.0
    U, s, V = Q.svd_rv_batch(F)
    Uo, so, Vo = O.svd_rv(F)
    rec = np.einsum("eab,eb,ecb->eac", U, s, V)
    print("svd: max|sigma-ref|", np.abs(s - so).max(), "recon", np.abs(rec - F).max(),
          "detU", np.abs(np.linalg.det(U) - 1).max(), "detV", np.abs(np.linalg.det(V) - 1).max())
    sc = scenes.CONFIGS[name](frames=frames)
    mat_o = omat(sc.material)
    t = time.time()
    osys = O.build(sc.verts, sc.tets, sc.density, mat_o, sc.h, sc.gravity, sc.fixed)
    print("oracle build", time.time() - t)
    mesh = Q.TetMesh(sc.verts, sc.tets, sc.density)
    t = time.time()
    gsys = Q.build_system(mesh, M.from_spec(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    print("gpu build", time.time() - t, gsys.factor_info())
    gsys.set_graph_mode(graph)
    # factor solve
    B = rng.standard_normal((gsys.free.size, 3))
    X = gsys.sysfact.solve(B)
    Xo = osys.factor.solve(B)
    print("solve rel err", np.abs(X - Xo).max() / np.abs(Xo).max())
    # objective / gradient at a random deformed state
    x = sc.verts + 0.01 * rng.standard_normal(sc.verts.shape)
    y = sc.verts.copy()
    st = Q.SimState(q_l=y, q_prev=y, y=y)
    g = Q.objective(gsys, st, x)
    go = O.objective(osys, y, x)
    gr = Q.gradient(gsys, st, x)
    gro = O.gradient(osys, y, x)
    print("objective rel", abs(g - go) / abs(go), "gradient rel", np.abs(gr - gro).max() / np.abs(gro).max())
    # frames
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    state = Q.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    oq_l, oq_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(frames):
        t0 = time.time()
        state, r = Q.simulate_frame(gsys, state, cfg)
        t1 = time.time()
        x_o, _, ro = O.simulate_frame(osys, oq_l, oq_prev, iterations=sc.iterations, m=sc.m)
        t2 = time.time()
        oq_prev, oq_l = oq_l, x_o
        dx = np.abs(state.q_l - x_o).max() / np.abs(x_o).max()
        dg = max(abs(a - b) / max(abs(b), 1e-30) for a, b in zip(r.g, ro.g))
        print(f"frame {f}: dx {dx:.3e} dg {dg:.3e} trials {r.ls_trials} vs {ro.ls_trials} "
              f"gpu {1000*(t1-t0):.2f} ms cpu {1000*(t2-t1):.1f} ms")
    print("g gpu", r.g[:4], "g cpu", ro.g[:4])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c1", int(sys.argv[2]) if len(sys.argv) > 2 else 3,
         (sys.argv[3] != "host") if len(sys.argv) > 3 else True)
