"""B200 path vs the reference goldens and the CPU oracle (run with -m gpu).

Tolerances (north_star): positions 1e-9 relative (fp64), per-iteration g
sequence 1e-10 relative, line-search trial counts identical.
"""
import os

import numpy as np
import pytest

import oracle.qnsim_oracle as O
import paper_1604_07378_b200 as Q
from paper_1604_07378_b200 import _lib, scenes
from paper_1604_07378_b200.materials import from_spec
from tests.helpers import FIX, TwistScene, golden, material_specs, oracle_material, read_csv

pytestmark = pytest.mark.gpu

X_TOL = 1e-9
G_TOL = 1e-10
MATS = ["neohookean", "stvk", "polynomial", "corotated", "mooney_rivlin", "spline", "poly_cubic"]


@pytest.fixture(scope="module", autouse=True)
def _gpu(built_lib):
    _lib.require_gpu()


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def build(sc, spec=None, **kw):
    mesh = Q.TetMesh(sc.verts, sc.tets, sc.density)
    return Q.build_system(mesh, from_spec(spec or sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed, **kw)


# ---- element level -----------------------------------------------------------

def test_svd_against_reference_golden():
    d = golden("svd_materials.npz")
    U, s, V = Q.svd_rv_batch(d["F"])
    np.testing.assert_allclose(s, d["sigma"], rtol=0, atol=1e-13)
    assert np.abs(np.linalg.det(U) - 1).max() < 1e-12 and np.abs(np.linalg.det(V) - 1).max() < 1e-12
    rec = np.einsum("eab,eb,ecb->eac", U, s, V)
    ok = np.abs(s).min(axis=1) > 1e-9  # away from the clamp, U diag(s) V^T reproduces F
    assert np.abs(rec[ok] - d["F"][ok]).max() < 1e-12
    # sign rule: s0 >= s1 >= |s2|, s2 < 0 iff det F < 0 (linalg.py:95-103)
    assert np.all(s[:, 0] >= s[:, 1] - 1e-14) and np.all(s[:, 1] >= np.abs(s[:, 2]) - 1e-14)
    detF = np.linalg.det(d["F"])
    nz = np.abs(detF) > 1e-20
    assert np.all((s[nz, 2] < 0) == (detF[nz] < 0))
    assert np.all(np.abs(s) >= 1e-10)


@pytest.mark.parametrize("name", MATS)
def test_material_eval_against_reference_golden(name):
    d = golden("svd_materials.npz")
    mat = from_spec(material_specs()[name])
    sig = d["mat_sigma"]
    e = Q.vl_energy_batch(mat, sig)
    t = Q.vl_stress_batch(mat, sig)
    np.testing.assert_allclose(e, d[f"{name}_energy"], rtol=1e-13, atol=1e-13 * max(1, np.abs(d[f"{name}_energy"]).max()))
    np.testing.assert_allclose(t, d[f"{name}_stress"], rtol=1e-13, atol=1e-13 * np.abs(d[f"{name}_stress"]).max())
    assert Q.estimate_stiffness(mat) == pytest.approx(float(d[f"{name}_k"]), rel=1e-13)


@pytest.mark.parametrize("name", MATS)
def test_element_group_seam_against_reference_golden(name):
    """GPU VLGroup.energy / add_gradient (dynamics.py:57-67) at a state with inverted tets."""
    d = golden("meshes_elements.npz")
    sc = scenes.c1()
    system = build(sc, material_specs()[name])
    grp = system.groups[0]
    x = d["c1_x"]
    assert grp.energy(x) == pytest.approx(float(d[f"c1_{name}_energy"]), rel=1e-12)
    g = np.zeros_like(x)
    grp.add_gradient(x, g)
    assert rel(g, d[f"c1_{name}_grad"]) <= 1e-11


def test_objective_gradient_against_oracle():
    sc = scenes.c2(frames=1)
    system = build(sc)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    rng = np.random.default_rng(3)
    y = sc.verts + 0.01 * rng.standard_normal(sc.verts.shape)
    x = sc.verts + 0.03 * rng.standard_normal(sc.verts.shape)
    st = Q.SimState(q_l=y, q_prev=y, y=y)
    assert Q.objective(system, st, x) == pytest.approx(O.objective(osys, y, x), rel=1e-12)
    assert rel(Q.gradient(system, st, x), O.gradient(osys, y, x)) <= 1e-12


# ---- factorisation -------------------------------------------------------------

@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_prefactored_solve_against_oracle(cfg):
    sc = scenes.CONFIGS[cfg](frames=1)
    system = build(sc)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    B = np.random.default_rng(1).standard_normal((system.free.size, 3))
    X = system.sysfact.solve(B)
    assert rel(X, osys.factor.solve(B)) <= 1e-12
    assert rel(osys.A_free @ X, B) <= 1e-12
    X2 = system.sysfact.solve(B)
    np.testing.assert_array_equal(X, X2)  # deterministic (no float atomics), linalg test :83-90


def test_factorization_api_dense_and_errors():
    rng = np.random.default_rng(2)
    M = rng.standard_normal((40, 40))
    A = M @ M.T + 40 * np.eye(40)
    F = Q.factorize_spd(A)
    B = rng.standard_normal((40, 5))
    np.testing.assert_allclose(A @ F.solve(B), B, atol=1e-10)
    v = rng.standard_normal(40)
    np.testing.assert_allclose(A @ F.solve(v), v, atol=1e-10)
    with pytest.raises(Q.FactorizationError):
        Q.factorize_spd(np.diag([1.0, -1.0, 2.0]))
    with pytest.raises(ValueError):
        F.solve(np.ones(39))


# ---- frames --------------------------------------------------------------------

def run_gpu(system, sc, frames, kind="lbfgs", targets=None, iterations=None):
    cfg = Q.SolverConfig(kind=kind, iterations=iterations or sc.iterations, m=sc.m)
    st = Q.SimState(q_l=np.array(sc.q_l), q_prev=np.array(sc.q_prev))
    out = []
    for f in range(frames):
        st, rec = Q.simulate_frame(system, st, cfg, fixed_targets=None if targets is None else targets(f))
        out.append((st.q_l.copy(), rec))
    return out


def test_c1_100_frames_against_reference_golden():
    """configs[0] as specified: 100 frames x 10 L-BFGS iterations vs the reference."""
    d = golden("frames_c1_lbfgs.npz")
    sc = scenes.c1()
    system = build(sc)
    res = run_gpu(system, sc, int(d["frames"]))
    for f, (x, rec) in enumerate(res):
        assert rel(rec.g, d["g"][f]) <= G_TOL, f
        assert list(rec.ls_trials) == list(d["trials"][f]), f
        np.testing.assert_array_equal(rec.alphas, d["alphas"][f])
        if f"x_{f}" in d:
            assert rel(x, d[f"x_{f}"]) <= X_TOL, f


def test_c1_pdqn_against_reference_golden():
    d = golden("frames_c1_pdqn.npz")
    sc = scenes.c1()
    system = build(sc)
    res = run_gpu(system, sc, int(d["frames"]), kind="pd_qn")
    for f, (x, rec) in enumerate(res):
        assert rel(rec.g, d["g"][f]) <= G_TOL
        assert list(rec.ls_trials) == list(d["trials"][f])
    assert rel(res[-1][0], d["x_9"]) <= X_TOL


@pytest.mark.parametrize("kind", ["lbfgs", "pd_qn"])
def test_twist_golden_csv_on_gpu(kind):
    """The reference's own golden trajectory, through the B200 path."""
    g_ref, tr_ref = read_csv(os.path.join(FIX, f"twist_{kind}.csv"))
    ts = TwistScene()
    mesh = Q.TetMesh(ts.verts, ts.tets, ts.density)
    system = Q.build_system(mesh, Q.make_builtin("neohookean", {"mu": ts.mu, "lambda": ts.lam}), h=ts.h,
                            gravity=ts.gravity, fixed=ts.fixed)
    cfg = Q.SolverConfig(kind=kind, iterations=ts.iterations, m=5)
    st = Q.SimState(q_l=ts.verts.copy(), q_prev=ts.verts.copy())
    for f in range(ts.frames):
        st, rec = Q.simulate_frame(system, st, cfg, fixed_targets=ts.targets(f))
        assert rel(rec.g, g_ref[f]) <= G_TOL, f
        assert list(rec.ls_trials) == list(tr_ref[f]), f
        np.testing.assert_allclose(st.q_l[ts.fixed], ts.targets(f), rtol=0, atol=0)


def test_c2_frame0_against_reference_golden():
    """configs[1] first frame vs the reference as-is (dense 15 360^2 Cholesky)."""
    path = os.path.join(os.path.dirname(__file__), "golden", "frames_c2_frame0.npz")
    if not os.path.exists(path):
        pytest.skip("c2 golden not generated (make_golden.py without --quick)")
    d = np.load(path)
    sc = scenes.c2()
    system = build(sc)
    (x, rec), = run_gpu(system, sc, 1)
    assert rel(rec.g, d["g"][0]) <= G_TOL
    assert list(rec.ls_trials) == list(d["trials"][0])
    assert rel(x, d["x_0"]) <= X_TOL


def test_c2_three_frames_against_oracle():
    sc = scenes.c2()
    system = build(sc)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    res = run_gpu(system, sc, 3)
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(3):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=sc.iterations, m=sc.m)
        q_prev, q_l = q_l, x
        assert rel(res[f][1].g, rec.g) <= G_TOL
        assert res[f][1].ls_trials == rec.ls_trials
        assert rel(res[f][0], x) <= X_TOL


def test_c3_frame_against_oracle():
    """configs[2] (375k tets, spline VL, twisted, both ends pinned), 1 frame x 10 its."""
    sc = scenes.c3(frames=1)
    system = build(sc)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    (xg, rg), = run_gpu(system, sc, 1)
    x, _, ro = O.simulate_frame(osys, sc.q_l.copy(), sc.q_prev.copy(), iterations=sc.iterations, m=sc.m)
    assert rel(rg.g, ro.g) <= G_TOL
    assert rg.ls_trials == ro.ls_trials
    assert rel(xg, x) <= X_TOL


def test_c4_batch_against_reference_golden():
    """configs[3]: 1024 instances in one batched system; checked instances vs the reference."""
    d = golden("frames_c4_subset.npz")
    sc = scenes.c4()
    mesh = Q.TetMesh(sc.verts, sc.tets, sc.density)
    system = Q.build_batch_system(mesh, [from_spec(s) for s in sc.batch_materials], h=sc.h, gravity=sc.gravity,
                                  fixed=sc.fixed)
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    st = Q.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    for f in range(3):
        st, recs = Q.simulate_frame(system, st, cfg)
        assert len(recs) == 1024
        for b in d["instances"]:
            assert rel(recs[b].g, d[f"i{b}_g"][f]) <= G_TOL
            assert recs[b].ls_trials == list(d[f"i{b}_trials"][f])
    for b in d["instances"]:
        assert rel(st.q_l[b], d[f"i{b}_x_2"]) <= X_TOL


# ---- PCG solve mode (configs[4]) -------------------------------------------------

@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_pcg_mode_against_oracle(cfg):
    """PCG (to 1e-13) in place of the prefactored solve reproduces the
    reference trajectory of the direct method within the parity tolerance."""
    sc = scenes.CONFIGS[cfg](frames=2)
    system = build(sc, solver="pcg", pcg_tol=1e-13)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    res = run_gpu(system, sc, 2)
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(2):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=sc.iterations, m=sc.m)
        q_prev, q_l = q_l, x
        assert rel(res[f][1].g, rec.g) <= G_TOL
        assert res[f][1].ls_trials == rec.ls_trials
        assert rel(res[f][0], x) <= X_TOL


def test_c5_scaled_down_pcg_against_oracle():
    """configs[4] material (NH + cubic) and solver (PCG to 1e-10, the BASELINE
    setting) on a 40x10x10 bar, held to the north_star bar: positions 1e-9,
    g 1e-10 (measured: ~5e-15 / ~1e-12, tools/c5_tol_sweep.py), same trials."""
    sc = scenes.c5(grid=(40, 10, 10), frames=1)
    system = build(sc, solver="pcg", pcg_tol=1e-10)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    (xg, rg), = run_gpu(system, sc, 1)
    x, _, ro = O.simulate_frame(osys, sc.q_l.copy(), sc.q_prev.copy(), iterations=sc.iterations, m=sc.m)
    assert rel(rg.g, ro.g) <= G_TOL
    assert rel(xg, x) <= X_TOL
    assert rg.ls_trials == ro.ls_trials


def test_c5_scaled_down_amg_against_oracle():
    """AMG-preconditioned CG (same 1e-10 tolerance) on the scaled configs[4]
    bar: the north_star bar (1e-9 positions, 1e-10 g), far fewer CG iterations."""
    sc = scenes.c5(grid=(40, 10, 10), frames=1)
    system = build(sc, solver="amg", pcg_tol=1e-10)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    run = Q.ResidentRun(system, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev),
                        Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
    rg = run.step(record=True)[0]
    xg = run.state().q_l
    x, _, ro = O.simulate_frame(osys, sc.q_l.copy(), sc.q_prev.copy(), iterations=sc.iterations, m=sc.m)
    assert rel(rg.g, ro.g) <= G_TOL
    assert rel(xg, x) <= X_TOL
    assert rg.ls_trials == ro.ls_trials
    assert 0 < run.last_cg_iterations <= 40 * sc.iterations
    info = system.amg_info()
    assert info["levels"] >= 2


@pytest.mark.parametrize("env", [{"QN_AMG_ZF": "0"}, {"QN_PCG_REC": "0"}, {"QN_AMG_TAIL_ROWS": "100000"},
                                 {"QN_AMG_SMALL_ROWS": "100000"}, {"QN_AMG_CSR_LANES": "16"}])
def test_amg_variants_agree_with_the_default(env, monkeypatch):
    """The AMG-PCG kernel variants behind the experiment knobs (fp64 z with the separate r.z kernel, the
    fused-p SpMV instead of the recurrence form, the small levels in one launch with grid barriers,
    other lane counts on the CSR levels) solve the same systems: same frame within the north_star
    bar, same line-search trials, CG iteration counts within one per solve."""
    sc = scenes.c5(grid=(100, 25, 25), frames=1)
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)

    def frame():
        system = build(sc, solver="amg", pcg_tol=1e-10)
        run = Q.ResidentRun(system, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev), cfg)
        rec = run.step(record=True)[0]
        return run.state().q_l, rec, run.last_cg_iterations, system.amg_info()["levels"]

    x0, r0, cg0, levels = frame()
    assert levels >= 3
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    x1, r1, cg1, _ = frame()
    assert rel(x1, x0) <= X_TOL and rel(r1.g, r0.g) <= G_TOL
    assert r1.ls_trials == r0.ls_trials
    assert abs(cg1 - cg0) <= sc.iterations


@pytest.mark.parametrize("graph", [True, False])
def test_amg_graph_and_host_loop_agree(graph):
    sc = scenes.c5(grid=(20, 6, 6), frames=1)
    s1 = build(sc, solver="amg", pcg_tol=1e-12)
    if not graph:
        s1.set_graph_mode(False)
    (x1, r1), = run_gpu(s1, sc, 1)
    s2 = build(sc, solver="pcg", pcg_tol=1e-12)
    (x2, r2), = run_gpu(s2, sc, 1)
    assert rel(x1, x2) <= 1e-9 and rel(r1.g, r2.g) <= 1e-10


# ---- semantics and edge cases (test_solvers.py / test_dynamics.py analogues) -----

def unit_tet_mesh():
    return Q.TetMesh(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]), np.array([[0, 1, 2, 3]]), 24.0)


def test_free_fall_identity_system():
    """No materials: A = I, one pd_qn iteration lands on y (test_solvers.py:355-361)."""
    mesh = unit_tet_mesh()
    system = Q.build_system(mesh, [], h=1.0, gravity=(0, 0, -9.8))
    q = mesh.vertices.copy()
    st2, rec = Q.simulate_frame(system, Q.SimState(q_l=q, q_prev=q), Q.SolverConfig(kind="pd_qn", iterations=1))
    np.testing.assert_allclose(st2.q_l, q + np.array([0.0, 0.0, -9.8]), atol=1e-12)
    # x starts at y, so the gradient is exactly zero: the ||g|| early-out records
    # (g_x, 0 trials, alpha 0) like solvers.py:292-298
    assert rec.ls_trials == [0] and rec.alphas == [0.0] and rec.g == [0.0]


def test_frame_at_rest_is_bitwise_stationary():
    """test_solvers.py:343-352"""
    mesh = Q.load_tet_mesh(os.path.join(FIX, "bar_small.node"), os.path.join(FIX, "bar_small.ele"), 1000.0)
    system = Q.build_system(mesh, Q.make_builtin("corotated", {"mu": 1e4, "lambda": 4e4}), gravity=(0, 0, 0))
    q = mesh.vertices.copy()
    st2, rec = Q.simulate_frame(system, Q.SimState(q_l=q, q_prev=q), Q.SolverConfig(kind="pd_qn", iterations=5))
    assert np.array_equal(st2.q_l, q)
    assert rec.g0 == pytest.approx(0.0, abs=1e-12)


def elastic_system():
    mesh = Q.load_tet_mesh(os.path.join(FIX, "bar_small.node"), os.path.join(FIX, "bar_small.ele"), 1000.0)
    fixed = np.nonzero(mesh.vertices[:, 0] < 1e-9)[0]
    return mesh, Q.build_system(mesh, Q.make_builtin("neohookean", {"mu": 1e4, "lambda": 4e4}), fixed=fixed)


def test_m0_lbfgs_equals_pdqn_bitwise():
    """test_solvers.py:121-130"""
    mesh, system = elastic_system()
    rng = np.random.default_rng(33)
    x0 = mesh.vertices + 0.03 * rng.standard_normal(mesh.vertices.shape)
    x0[system.fixed] = mesh.vertices[system.fixed]
    st = Q.SimState(q_l=x0, q_prev=x0)
    a, ra = Q.simulate_frame(system, st.copy(), Q.SolverConfig(kind="lbfgs", m=0, iterations=6))
    b, rb = Q.simulate_frame(system, st.copy(), Q.SolverConfig(kind="pd_qn", iterations=6))
    np.testing.assert_array_equal(a.q_l, b.q_l)
    assert ra.g == rb.g


def test_monotone_objective_and_record_shapes():
    mesh, system = elastic_system()
    rng = np.random.default_rng(33)
    x0 = mesh.vertices + 0.03 * rng.standard_normal(mesh.vertices.shape)
    x0[system.fixed] = mesh.vertices[system.fixed]
    for kind in ("pd_qn", "lbfgs"):
        _, rec = Q.simulate_frame(system, Q.SimState(q_l=x0, q_prev=x0), Q.SolverConfig(kind=kind, iterations=7))
        gs = [rec.g0] + rec.g
        assert all(b <= a + 1e-12 * max(abs(a), 1.0) for a, b in zip(gs, gs[1:])), kind
        assert len(rec.g) == len(rec.ls_trials) == len(rec.cum_ms) == len(rec.alphas) == 7
        assert all(b >= a for a, b in zip(rec.cum_ms, rec.cum_ms[1:]))


def test_fixed_targets_enforced():
    """test_solvers.py:388-395"""
    mesh, system = elastic_system()
    q = mesh.vertices.copy()
    targets = q[system.fixed] + np.array([0.0, 0.0, 0.01])
    st2, _ = Q.simulate_frame(system, Q.SimState(q_l=q, q_prev=q), Q.SolverConfig(kind="lbfgs"),
                              fixed_targets=targets)
    assert np.allclose(st2.q_l[system.fixed], targets)


def test_no_line_search_mode_against_oracle():
    mesh, system = elastic_system()
    osys = O.build(mesh.vertices, mesh.tets, 1000.0, O.builtin("neohookean", mu=1e4, lam=4e4), system.h,
                   (0, 0, -9.8), system.fixed, factor="dense")
    q = mesh.vertices.copy()
    st2, rec = Q.simulate_frame(system, Q.SimState(q_l=q, q_prev=q),
                                Q.SolverConfig(kind="lbfgs", iterations=5, line_search=False))
    x, _, ro = O.simulate_frame(osys, q, q, iterations=5, use_line_search=False)
    assert rel(st2.q_l, x) <= X_TOL and rel(rec.g, ro.g) <= G_TOL
    assert rec.ls_trials == [1] * 5 and rec.alphas == [1.0] * 5


def test_deterministic_and_graph_equals_host_loop():
    sc = scenes.c1(frames=2)
    a = build(sc)
    b = build(sc)
    b.set_graph_mode(False)
    ra = run_gpu(a, sc, 2)
    rb = run_gpu(b, sc, 2)
    rc = run_gpu(a, sc, 2)
    for (xa, ga), (xb, gb), (xc, gc) in zip(ra, rb, rc):
        np.testing.assert_array_equal(xa, xb)
        np.testing.assert_array_equal(xa, xc)
        assert ga.g == gb.g == gc.g


def test_unsupported_options_raise():
    sc = scenes.c1(frames=1)
    system = build(sc)
    st = Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev)
    cs = Q.build_system(Q.TetMesh(sc.verts, sc.tets), from_spec(sc.material), fixed=sc.fixed,
                        colliders=[Q.dynamics.HalfSpace((0, 0, -1), (0, 0, 1))])
    with pytest.raises(NotImplementedError):
        Q.simulate_frame(cs, st, Q.SolverConfig(kind="newton"))
    with pytest.raises(Q.DynamicsError):
        Q.build_system(Q.TetMesh(sc.verts, sc.tets), from_spec(sc.material), fixed=np.arange(sc.verts.shape[0]))


def test_resident_run_matches_stateless():
    sc = scenes.c1(frames=3)
    s1 = build(sc)
    res = run_gpu(s1, sc, 3)
    s2 = build(sc)
    run = Q.ResidentRun(s2, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev), Q.SolverConfig(kind="lbfgs"))
    for f in range(3):
        recs = run.step(record=True)
        assert recs[0].g == res[f][1].g
    np.testing.assert_array_equal(run.state().q_l, res[-1][0])
    assert run.last_ms > 0 and run.last_passes >= 10


@pytest.mark.gpu
def test_pinned_out_buffers_bitwise_equal():
    import torch
    sc = scenes.c1(frames=2)
    s1 = build(sc)
    res = run_gpu(s1, sc, 2)
    s2 = build(sc)
    keep = [torch.empty(np.asarray(sc.q_l).shape, dtype=torch.float64, pin_memory=True) for _ in range(4)]
    h = [k.numpy() for k in keep]
    h[0][...] = sc.q_l
    h[1][...] = sc.q_prev
    st = Q.SimState(q_l=h[0], q_prev=h[1])
    for f, slot in enumerate((2, 1)):
        st, rec = Q.simulate_frame(s2, st, Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m), out=Q.SimState(q_l=h[slot], q_prev=None, y=h[3]))
        assert st.q_l is h[slot]
        np.testing.assert_array_equal(st.q_l, res[f][0])
    with pytest.raises(ValueError):
        Q.simulate_frame(s2, st, Q.SolverConfig(kind="lbfgs"), out=Q.SimState(q_l=np.zeros(3), q_prev=None, y=h[3]))


def test_torch_custom_ops_match_the_c_abi_paths():
    import torch
    from paper_1604_07378_b200 import torch_ops
    d = golden("svd_materials.npz")
    F = torch.from_numpy(d["F"]).cuda()
    U, s, V = torch.ops.qnsim_b200.svd_rv(F)
    Ur, sr, Vr = Q.svd_rv_batch(d["F"])
    assert np.array_equal(s.cpu().numpy(), sr) and np.array_equal(U.cpu().numpy(), Ur)
    sc = scenes.c1(frames=1)
    system = build(sc)
    B = np.random.default_rng(4).standard_normal((system.sysfact.n, 3))
    X = torch.ops.qnsim_b200.factor_solve(system.sysfact.op_handle, torch.from_numpy(B).cuda(), 0)
    np.testing.assert_array_equal(X.cpu().numpy(), system.sysfact.solve(B))
    y = np.asarray(sc.q_l) + 0.01
    g, grad = torch.ops.qnsim_b200.objective(system.op_handle, torch.from_numpy(np.asarray(sc.q_l)).cuda(),
                                             torch.from_numpy(y).cuda())
    g_ref = Q.objective(system, Q.SimState(q_l=np.asarray(sc.q_l), q_prev=np.asarray(sc.q_prev), y=y),
                        np.asarray(sc.q_l))
    assert float(g.cpu()[0]) == pytest.approx(g_ref, rel=1e-13)
    run = Q.ResidentRun(system, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev),
                        Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
    gs, status = torch.ops.qnsim_b200.frame_step(system.op_handle, 1, sc.iterations, sc.m, 1)
    assert gs.is_cuda and status.is_cuda  # device-only: no host round trip inside the op
    (_, rec), = run_gpu(build(sc), sc, 1)
    np.testing.assert_array_equal(gs.cpu().numpy()[0], np.asarray(rec.g))
    assert int(status.cpu()[0]) == 0
    # the objective op runs in order on torch's current stream: inputs produced
    # by a kernel just before the call on the same stream are seen complete
    xq = torch.from_numpy(np.asarray(sc.q_l)).cuda()
    for _ in range(3):
        x2 = xq * 1.0 + 0.0
        y2 = x2 + 0.01
        g2, _ = torch.ops.qnsim_b200.objective(system.op_handle, x2, y2)
        assert float(g2.cpu()[0]) == pytest.approx(g_ref, rel=1e-13)
    h = torch_ops.register_material(from_spec(sc.material))
    psi, tau = torch.ops.qnsim_b200.material_eval(h, s[:16].contiguous())
    assert psi.shape == (16,) and tau.shape == (16, 3)


# ---- analogues of the reference's unit edge cases (test_linalg / test_dynamics) ----

def test_svd_rv_edge_cases_like_reference():
    # identity, diagonal, reflection onto the last sigma, clamp of singular input (test_linalg.py:93-147)
    r = Q.svd_rv(np.eye(3))
    np.testing.assert_allclose(r.sigma, [1, 1, 1], atol=1e-15)
    r = Q.svd_rv(np.diag([3.0, 2.0, 1.0]))
    np.testing.assert_allclose(r.sigma, [3, 2, 1], atol=1e-14)
    r = Q.svd_rv(np.diag([2.0, 1.0, -3.0]))  # det < 0: the sign goes to the smallest |sigma|
    assert r.sigma[2] < 0 and np.all(r.sigma[:2] > 0)
    assert np.linalg.det(r.U) == pytest.approx(1.0) and np.linalg.det(r.V) == pytest.approx(1.0)
    r = Q.svd_rv(np.zeros((3, 3)))
    assert np.all(np.abs(r.sigma) >= 1e-10 - 1e-25)
    with pytest.raises(ValueError):
        Q.svd_rv(np.full((3, 3), np.nan))
    with pytest.raises(ValueError):
        Q.svd_rv(np.zeros((2, 3)))


def test_objective_zero_at_rest_and_fixed_rows_and_translation():
    # test_dynamics.py:149 (zero at rest), :233 (fixed rows zero), :243 (elastic forces sum to zero)
    sc = scenes.c1(frames=1)
    system = build(sc)
    x0 = np.asarray(sc.verts)
    st = Q.SimState(q_l=x0, q_prev=x0, y=x0)
    assert abs(Q.objective(system, st, x0)) <= 1e-9 * max(1.0, np.abs(x0).max())
    rng = np.random.default_rng(7)
    x = x0 + 0.02 * rng.standard_normal(x0.shape)
    g = Q.gradient(system, st, x)
    assert np.all(g[sc.fixed] == 0.0)
    # elastic part of the gradient (inertia removed via y = x) sums to zero over all vertices
    free_sys = build(sc, **{})
    st_x = Q.SimState(q_l=x, q_prev=x, y=x)
    ge = Q.gradient(Q.build_system(Q.TetMesh(sc.verts, sc.tets, sc.density), from_spec(sc.material), h=sc.h,
                                   gravity=sc.gravity, fixed=()), st_x, x)
    assert np.abs(ge.sum(axis=0)).max() <= 1e-9 * np.abs(ge).max()
    del free_sys


def test_factorize_rejects_nonsquare_and_solve_dimension_mismatch():
    # test_linalg.py:48-81: nonsquare -> FactorizationError, row mismatch -> ValueError
    with pytest.raises(Q.FactorizationError):
        Q.factorize_spd(np.ones((3, 4)))
    F = Q.factorize_spd(np.eye(4) * 2.0)
    np.testing.assert_allclose(Q.solve_prefactored(F, np.ones((4, 3))), 0.5 * np.ones((4, 3)), rtol=0, atol=1e-15)
    F1 = Q.factorize_spd(np.array([[4.0]]))
    np.testing.assert_allclose(Q.solve_prefactored(F1, np.array([[8.0, 4.0, 0.0]])), [[2.0, 1.0, 0.0]], atol=1e-15)
    with pytest.raises(ValueError):
        Q.solve_prefactored(F, np.ones((5, 3)))


def test_factorization_reuse_bit_identical():
    sc = scenes.c2(frames=1)
    system = build(sc)
    B = np.random.default_rng(8).standard_normal((system.sysfact.n, 3))
    X1 = system.sysfact.solve(B)
    X2 = system.sysfact.solve(B)
    assert np.array_equal(X1, X2)


# ---- colliders -----------------------------------------------

def _gpu_collider_run(sc, cols, frames, collision_weight=None, graph=True):
    from tests.helpers import make_colliders
    from paper_1604_07378_b200 import dynamics as D
    system = build(sc, colliders=make_colliders(cols, D), collision_weight=collision_weight)
    if not graph:
        system.set_graph_mode(False)
    return system, run_gpu(system, sc, frames)


@pytest.mark.parametrize("graph", [True, False])
def test_colliders_three_kinds_against_reference_golden(graph):
    """Half-space, sphere and torus penalties (update_collisions every
    iteration, dynamics.py:486-516) inside the frame graph: the reference's
    own trajectory (tests/golden/frames_collider_bar.npz)."""
    from tests.helpers import collider_bar_scene
    sc, cols = collider_bar_scene()
    d = golden("frames_collider_bar.npz")
    system, res = _gpu_collider_run(sc, cols, int(d["frames"]), graph=graph)
    assert system.w_col == float(d["w_col"])
    for f, (x, rec) in enumerate(res):
        assert rel(rec.g, d["g"][f]) <= G_TOL
        assert rec.ls_trials == list(d["trials"][f])
        if f"x_{f}" in d:
            assert rel(x, d[f"x_{f}"]) <= X_TOL


def test_sphere_drop_scenario_against_reference_harness():
    """The reference's bundled sphere_drop.json scenario, 30 frames.  Penalty
    contact amplifies roundoff through active-set flips: the reference itself,
    run with its tet list reversed (same mathematics, another summation
    order), departs from its own trajectory by 1e-12 at frame 2 and by ~4e-2
    in g / ~5e-4 in x once the sphere rests on the floor (golden rev_*).  The
    B200 run must match strictly until contact and stay inside 4x that
    envelope after it."""
    from tests.helpers import SphereDropScene
    sd = SphereDropScene()
    d = golden("frames_sphere_drop.npz")
    _, res = _gpu_collider_run(sd, sd.cols, int(d["frames"]), collision_weight=sd.collision_weight)
    g_ref, g_rev = d["g"], d["rev_g"]
    env_g = max(np.abs(g_rev[f] - g_ref[f]).max() / np.abs(g_ref[f]).max() for f in range(2, g_ref.shape[0]))
    env_x = max(rel(d[f"rev_x_{f}"], d[f"x_{f}"]) for f in (9, 19, 29))
    for f, (x, rec) in enumerate(res):
        if f <= 3:  # before contact: the strict parity bar
            np.testing.assert_allclose(rec.g, g_ref[f], rtol=G_TOL, atol=1e-12)
            assert rec.ls_trials == list(d["trials"][f])
        else:
            assert np.abs(np.array(rec.g) - g_ref[f]).max() / np.abs(g_ref[f]).max() <= 4 * env_g
        if f"x_{f}" in d:
            assert rel(x, d[f"x_{f}"]) <= (X_TOL if f == 0 else 4 * env_x)


def test_colliders_batch_instances_match_single():
    """Batched instances (configs[3] machinery) with colliders: identical
    instances stay bitwise identical, and equal the single-system run within
    the parity tolerance (the batched solve sums in another order)."""
    from tests.helpers import collider_bar_scene, make_colliders
    from paper_1604_07378_b200 import dynamics as D
    sc, cols = collider_bar_scene()
    mesh = Q.TetMesh(sc.verts, sc.tets, sc.density)
    mat = from_spec(sc.material)
    bsys = Q.build_batch_system(mesh, [mat, mat, mat], h=sc.h, gravity=sc.gravity, fixed=sc.fixed,
                                colliders=make_colliders(cols, D))
    ssys = build(sc, colliders=make_colliders(cols, D))
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    bst = Q.SimState(q_l=np.stack([sc.q_l] * 3), q_prev=np.stack([sc.q_prev] * 3))
    sst = Q.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    for _ in range(3):
        bst, brecs = Q.simulate_frame(bsys, bst, cfg)
        sst, srec = Q.simulate_frame(ssys, sst, cfg)
        for b in range(3):
            assert np.array_equal(bst.q_l[b], bst.q_l[0]) and brecs[b].g == brecs[0].g
            assert rel(bst.q_l[b], sst.q_l) <= X_TOL and rel(brecs[b].g, srec.g) <= G_TOL
            assert brecs[b].ls_trials == srec.ls_trials


@pytest.mark.parametrize("name", ["arap", "mixed"])
def test_arap_groups_against_reference_golden(name):
    """PDMaterial("arap") tets (dynamics.ARAPGroup, dynamics.py:73-108) run as
    the Valanis-Landel material k/2 (s - 1)^2 with w = vol k, alone and
    alternating with a Neo-Hookean group: 10 frames vs the reference."""
    from paper_1604_07378_b200.materials import PDMaterial
    sc = scenes.c1(grid=(10, 3, 3), iterations=10)
    d = golden("frames_arap.npz")
    half = np.arange(sc.tets.shape[0]) % 2 == 0
    mats = PDMaterial("arap", 2e5) if name == "arap" else \
        [(np.nonzero(half)[0], PDMaterial("arap", 2e5)), (np.nonzero(~half)[0], from_spec(sc.material))]
    system = Q.build_system(Q.TetMesh(sc.verts, sc.tets, sc.density), mats, h=sc.h, gravity=sc.gravity,
                            fixed=sc.fixed)
    res = run_gpu(system, sc, 10)
    for f, (x, rec) in enumerate(res):
        assert rel(rec.g, d[f"{name}_g"][f]) <= G_TOL
        assert rec.ls_trials == list(d[f"{name}_trials"][f])
    assert rel(res[-1][0], d[f"{name}_x_9"]) <= X_TOL


@pytest.mark.parametrize("name", ["default", "aggressive"])
@pytest.mark.parametrize("graph", [True, False])
def test_chebyshev_against_reference_golden(name, graph):
    """kind="chebyshev": omega schedule, x_prev_iter bookkeeping and the
    non-descent fallback (rec.fallbacks) on the device, vs the reference."""
    sc = scenes.c2(grid=(12, 3, 3), iterations=20)
    d = golden("frames_chebyshev.npz")
    system = build(sc)
    if not graph:
        system.set_graph_mode(False)
    cfg = Q.SolverConfig(kind="chebyshev", iterations=sc.iterations, rho=float(d[f"{name}_rho"]),
                         S=int(d[f"{name}_S"]))
    st = Q.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    for f in range(8):
        st, rec = Q.simulate_frame(system, st, cfg)
        assert rel(rec.g, d[f"{name}_g"][f]) <= G_TOL
        assert rec.ls_trials == list(d[f"{name}_trials"][f])
        assert rec.fallbacks == int(d[f"{name}_fallbacks"][f])
    assert rel(st.q_l, d[f"{name}_x_7"]) <= X_TOL


@pytest.mark.parametrize("graph", [True, False])
def test_lbfgs_scaled_identity_against_reference_golden(graph):
    """lbfgs_init="scaled_identity": the two-loop with H0 = rho/<t,t> I (no
    solve) on the device, vs the reference."""
    sc = scenes.c2(grid=(12, 3, 3), iterations=20)
    d = golden("frames_chebyshev.npz")
    system = build(sc)
    if not graph:
        system.set_graph_mode(False)
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m, lbfgs_init="scaled_identity")
    st = Q.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    # frames of this method end unconverged and pass their roundoff on,
    # amplified: the reference with its tet list reversed departs from itself
    # by 4e-10 in g at frame 3 and 6e-4 at frame 7 (golden scaled_rev_*).
    # The bar: the strict tolerance, or 10x that envelope once it exceeds it
    # (a single reordering samples the envelope; the device rounds differently).
    env = [np.abs(d["scaled_rev_g"][f] - d["scaled_g"][f]).max() / np.abs(d["scaled_g"][f]).max() for f in range(8)]
    for f in range(8):
        st, rec = Q.simulate_frame(system, st, cfg)
        assert rel(rec.g, d["scaled_g"][f]) <= max(G_TOL, 10 * max(env[: f + 1]))
        if env[f] < 1e-12:
            assert rec.ls_trials == list(d["scaled_trials"][f])
    assert rel(st.q_l, d["scaled_x_7"]) <= 10 * rel(d["scaled_rev_x_7"], d["scaled_x_7"])
    # switching back to the system-matrix init rebuilds the graph
    st2, rec2 = Q.simulate_frame(system, Q.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy()),
                                 Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
    assert rec2.ls_trials[0] == 1


@pytest.mark.parametrize("graph", [True, False])
def test_cloth_hang_scenario_against_reference_harness(graph):
    """Spring networks (cloth): the reference's cloth_hang.json, 20 frames."""
    from paper_1604_07378_b200.materials import PDMaterial
    from tests.helpers import ClothScene
    cs = ClothScene()
    d = golden("frames_cloth_hang.npz")
    mesh = Q.load_obj_springs(os.path.join(FIX, "cloth20.obj"), density=cs.density)
    assert np.array_equal(mesh.edges, cs.edges)
    system = Q.build_system(mesh, PDMaterial("mass_spring", cs.k), h=cs.h, gravity=cs.gravity, fixed=cs.fixed)
    if not graph:
        system.set_graph_mode(False)
    res = run_gpu(system, cs, int(d["frames"]))
    for f, (x, rec) in enumerate(res):
        assert rel(rec.g, d["g"][f]) <= G_TOL
        assert rec.ls_trials == list(d["trials"][f])
        if f"x_{f}" in d:
            assert rel(x, d[f"x_{f}"]) <= X_TOL


@pytest.mark.parametrize("name", ["uniform", "two"])
def test_aniso_fibres_against_reference_golden(name):
    """Anisotropic fibres (dynamics.AnisoGroup) on the fibre branch of the
    per-tet kernel, appended after the Neo-Hookean group: 10 frames."""
    from tests.helpers import aniso_cases
    sc = scenes.c1(grid=(10, 3, 3), iterations=10)
    d = golden("frames_aniso.npz")
    system = build(sc, aniso=aniso_cases(sc.tets.shape[0])[name])
    res = run_gpu(system, sc, 10)
    for f, (x, rec) in enumerate(res):
        assert rel(rec.g, d[f"{name}_g"][f]) <= G_TOL
        assert rec.ls_trials == list(d[f"{name}_trials"][f])
    assert rel(res[-1][0], d[f"{name}_x_9"]) <= X_TOL


def test_newton_frames_and_reference_minimum_against_reference():
    """kind="newton" and newton_reference on the device (central-difference
    element Hessians, eigenvalue floor, dense Cholesky): frames vs the
    reference within the finite-difference noise (see the oracle test), the
    reference minimum g* of configs[0]'s first frame to 1e-12."""
    d = golden("frames_newton.npz")
    sc = scenes.c2(grid=(6, 2, 2), iterations=5)
    system = build(sc)
    st = Q.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    for f in range(3):
        st, rec = Q.simulate_frame(system, st, Q.SolverConfig(kind="newton", iterations=sc.iterations))
        assert rel(rec.g, d["frames_g"][f]) <= G_TOL  # measured ~7e-12
        assert rec.ls_trials == list(d["frames_trials"][f])
    assert rel(st.q_l, d["frames_x_2"]) <= X_TOL
    sc1 = scenes.c1()
    s1 = build(sc1)
    xs, gs = Q.newton_reference(s1, Q.SimState(q_l=sc1.q_l.copy(), q_prev=sc1.q_prev.copy()))
    assert abs(gs - float(d["c1_gstar"])) <= 1e-12 * abs(gs)  # measured 8e-14
    assert rel(xs, d["c1_xstar"]) <= 1e-9


def test_lbfgs_rest_pose_hessian_against_reference_golden():
    """lbfgs_init="rest_pose_hessian": the Newton Hessian at rest, factored and
    inverted once on the device, applied in the frame graph's direction step."""
    d = golden("frames_newton.npz")
    sc = scenes.c2(grid=(6, 2, 2), iterations=10)
    system = build(sc)
    st = Q.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    cfg = Q.SolverConfig(kind="lbfgs", iterations=10, m=5, lbfgs_init="rest_pose_hessian")
    # the frames converge to roundoff within the budget: decisions at the
    # noise floor depend on summation order, so the bar is the strict one or
    # 10x the reference's own reordering envelope (golden rest_rev_*)
    for f in range(3):
        st, rec = Q.simulate_frame(system, st, cfg)
        env = np.abs(d["rest_rev_g"][f] - d["rest_g"][f]).max() / np.abs(d["rest_g"][f]).max()
        assert rel(rec.g, d["rest_g"][f]) <= max(G_TOL, 10 * env)
    assert rel(st.q_l, d["rest_x_2"]) <= max(X_TOL, 10 * rel(d["rest_rev_x_2"], d["rest_x_2"]))


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_fp32_element_pass_within_the_fp32_tolerance(cfg):
    """The optional fp32 mode (configs[2] "optional fp32 run", north star: 1e-4
    on positions): the per-tet pass in single precision, everything else fp64,
    vs the fp64 oracle on scaled configs (StVK with initial velocity; the
    seeded Hermite-spline material with both ends pinned)."""
    sc = scenes.c2(grid=(20, 5, 5), frames=3) if cfg == "c2" else scenes.c3(grid=(20, 5, 5), frames=3)
    system = build(sc, precision="fp32")
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    res = run_gpu(system, sc, 3)
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(3):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=sc.iterations, m=sc.m)
        q_prev, q_l = q_l, x
        # positions: the north-star fp32 bar; energies carry the fp32
        # evaluation of expanded polynomials (StVK terms cancel to ~1e-7 of
        # their 4e5 magnitude), an offset of ~1e-4 of g0
        assert rel(res[f][0], x) <= 1e-4
        assert rel(res[f][1].g, rec.g) <= 1e-3
