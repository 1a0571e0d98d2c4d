"""Pin the CPU oracle to the reference: golden vectors written by the
unmodified reference (tests/golden/make_golden.py) and the reference's own
golden trajectories twist_{lbfgs,pd_qn}.csv."""
import numpy as np
import pytest

import oracle.qnsim_oracle as O
from paper_1604_07378_b200 import scenes
import os

from tests.helpers import FIX, TwistScene, golden, material_specs, oracle_material, read_csv

MATS = ["neohookean", "stvk", "polynomial", "corotated", "mooney_rivlin", "spline", "poly_cubic"]


def test_svd_matches_reference():
    d = golden("svd_materials.npz")
    U, s, V = O.svd_rv(d["F"])
    np.testing.assert_allclose(s, d["sigma"], rtol=0, atol=1e-13)
    assert np.all(np.abs(np.linalg.det(U) - 1) < 1e-12) and np.all(np.abs(np.linalg.det(V) - 1) < 1e-12)


@pytest.mark.parametrize("name", MATS)
def test_materials_match_reference(name):
    d = golden("svd_materials.npz")
    mat = oracle_material(material_specs()[name])
    sig = d["mat_sigma"]
    e, t = O.vl_energy(mat, sig), O.vl_stress(mat, sig)
    scale = max(1.0, np.abs(d[f"{name}_energy"]).max())
    np.testing.assert_allclose(e, d[f"{name}_energy"], rtol=1e-13, atol=1e-13 * scale)
    np.testing.assert_allclose(t, d[f"{name}_stress"], rtol=1e-13, atol=1e-13 * np.abs(d[f"{name}_stress"]).max())
    assert mat.shift == pytest.approx(float(d[f"{name}_shift"]), rel=1e-15, abs=1e-12)
    assert O.fit_stiffness(mat) == pytest.approx(float(d[f"{name}_k"]), rel=1e-13)


def test_grid_bar_matches_reference_bar_mesh():
    d = golden("meshes_elements.npz")
    for key, args in {"bar_c1": (20, 5, 5, (2.0, 0.5, 0.5)), "bar_small": (6, 2, 2, (0.6, 0.2, 0.2))}.items():
        v, t = O.grid_bar(*args)
        np.testing.assert_array_equal(t, d[f"{key}_tets"])
        np.testing.assert_array_equal(v, d[f"{key}_verts"])
    sc = scenes.c1()
    np.testing.assert_array_equal(O.vertex_masses(sc.verts, sc.tets, 1000.0), d["c1_masses"])


@pytest.mark.parametrize("name", MATS)
def test_element_energy_gradient_match_reference(name):
    d = golden("meshes_elements.npz")
    sc = scenes.c1()
    mat = oracle_material(material_specs()[name])
    G, vols = O.diff_operators(sc.verts, sc.tets)
    grp = O.TetGroup(sc.tets, G, vols, mat, 1.0)
    x = d["c1_x"]
    e = grp.energy(x)
    assert e == pytest.approx(float(d[f"c1_{name}_energy"]), rel=1e-12)
    g = np.zeros_like(x)
    grp.add_gradient(x, g)
    ref = d[f"c1_{name}_grad"]
    assert np.abs(g - ref).max() <= 1e-11 * np.abs(ref).max()


def test_c1_frames_match_reference():
    d = golden("frames_c1_lbfgs.npz")
    sc = scenes.c1()
    sysm = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                   factor="dense")
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    n = 20
    for f in range(n):
        x, _, rec = O.simulate_frame(sysm, q_l, q_prev, iterations=sc.iterations, m=sc.m)
        q_prev, q_l = q_l, x
        np.testing.assert_allclose(rec.g, d["g"][f], rtol=1e-11)
        assert list(rec.ls_trials) == list(d["trials"][f])
        if f"x_{f}" in d:
            assert np.abs(x - d[f"x_{f}"]).max() <= 1e-12 * np.abs(d[f"x_{f}"]).max()


def test_c1_pdqn_frames_match_reference():
    d = golden("frames_c1_pdqn.npz")
    sc = scenes.c1()
    sysm = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                   factor="dense")
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(int(d["frames"])):
        x, _, rec = O.simulate_frame(sysm, q_l, q_prev, iterations=sc.iterations, m=sc.m, kind="pd_qn")
        q_prev, q_l = q_l, x
        np.testing.assert_allclose(rec.g, d["g"][f], rtol=1e-11)
        assert list(rec.ls_trials) == list(d["trials"][f])


@pytest.mark.parametrize("kind", ["lbfgs", "pd_qn"])
def test_twist_golden_csv(kind):
    """The reference's own golden trajectory (frontend/tests/fixtures/twist_*.csv)."""
    g_ref, tr_ref = read_csv(os.path.join(FIX, f"twist_{kind}.csv"))
    ts = TwistScene()
    mat = O.builtin("neohookean", mu=ts.mu, lam=ts.lam)
    sysm = O.build(ts.verts, ts.tets, ts.density, mat, ts.h, ts.gravity, ts.fixed, factor="dense")
    q_l = ts.verts.copy()
    q_prev = ts.verts.copy()
    for f in range(ts.frames):
        x, _, rec = O.simulate_frame(sysm, q_l, q_prev, iterations=ts.iterations, m=5, kind=kind,
                                     fixed_targets=ts.targets(f))
        q_prev, q_l = q_l, x
        np.testing.assert_allclose(rec.g, g_ref[f], rtol=1e-12)
        assert list(rec.ls_trials) == list(tr_ref[f])


def test_c4_subset_matches_reference():
    d = golden("frames_c4_subset.npz")
    sc = scenes.c4()
    for b in d["instances"]:
        sysm = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.batch_materials[b]), sc.h, sc.gravity,
                       sc.fixed, factor="dense")
        q_l, q_prev = sc.verts.copy(), sc.verts.copy()
        for f in range(3):
            x, _, rec = O.simulate_frame(sysm, q_l, q_prev, iterations=sc.iterations, m=sc.m)
            q_prev, q_l = q_l, x
            np.testing.assert_allclose(rec.g, d[f"i{b}_g"][f], rtol=1e-11)
        assert np.abs(x - d[f"i{b}_x_2"]).max() <= 1e-12 * np.abs(x).max()


def test_sparse_factor_equals_dense():
    sc = scenes.c1()
    mat = oracle_material(sc.material)
    a = O.build(sc.verts, sc.tets, sc.density, mat, sc.h, sc.gravity, sc.fixed, factor="dense")
    b = O.build(sc.verts, sc.tets, sc.density, mat, sc.h, sc.gravity, sc.fixed, factor="sparse")
    B = np.random.default_rng(0).standard_normal((a.free.size, 3))
    xa, xb = a.factor.solve(B), b.factor.solve(B)
    assert np.abs(xa - xb).max() <= 1e-13 * np.abs(xa).max()


# ---- colliders: oracle vs the reference's own runs ----------

def _collider_frames(sys_, sc, frames):
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(frames):
        x, _, rec = O.simulate_frame(sys_, q_l, q_prev, iterations=sc.iterations, m=sc.m)
        q_prev, q_l = q_l, x
        yield f, x, rec


def test_oracle_colliders_three_kinds_match_reference():
    from tests.helpers import collider_bar_scene, make_colliders
    sc, cols = collider_bar_scene()
    d = golden("frames_collider_bar.npz")
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                   factor="dense", colliders=make_colliders(cols, O))
    assert osys.w_col == float(d["w_col"])
    for f, x, rec in _collider_frames(osys, sc, 10):
        np.testing.assert_allclose(rec.g, d["g"][f], rtol=1e-12)
        assert list(rec.ls_trials) == list(d["trials"][f])
        if f"x_{f}" in d:
            np.testing.assert_allclose(x, d[f"x_{f}"], rtol=0, atol=1e-12 * np.abs(d[f"x_{f}"]).max())


def test_oracle_sphere_drop_matches_reference_harness():
    from tests.helpers import SphereDropScene, make_colliders
    sd = SphereDropScene()
    d = golden("frames_sphere_drop.npz")
    osys = O.build(sd.verts, sd.tets, sd.density, oracle_material(sd.material), sd.h, sd.gravity, sd.fixed,
                   factor="dense", colliders=make_colliders(sd.cols, O), collision_weight=sd.collision_weight)
    for f, x, rec in _collider_frames(osys, sd, 10):  # contact starts at frame ~7
        np.testing.assert_allclose(rec.g, d["g"][f], rtol=1e-12, atol=1e-12)
        assert list(rec.ls_trials) == list(d["trials"][f])
        if f"x_{f}" in d:
            np.testing.assert_allclose(x, d[f"x_{f}"], rtol=0, atol=1e-12 * np.abs(d[f"x_{f}"]).max())


def _arap_case(name, sc):
    m = sc.tets.shape[0]
    half = np.arange(m) % 2 == 0
    if name == "arap":
        return O.ARAP(2e5)
    return [(np.nonzero(half)[0], O.ARAP(2e5)), (np.nonzero(~half)[0], oracle_material(sc.material))]


@pytest.mark.parametrize("name", ["arap", "mixed"])
def test_oracle_arap_groups_match_reference(name):
    """PDMaterial("arap") tets alone and mixed with a VL group (dynamics.py:73-108, 330-345)."""
    sc = scenes.c1(grid=(10, 3, 3), iterations=10)
    d = golden("frames_arap.npz")
    osys = O.build(sc.verts, sc.tets, sc.density, _arap_case(name, sc), sc.h, sc.gravity, sc.fixed, factor="dense")
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(10):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=sc.iterations, m=sc.m)
        q_prev, q_l = q_l, x
        np.testing.assert_allclose(rec.g, d[f"{name}_g"][f], rtol=1e-12)
        assert list(rec.ls_trials) == list(d[f"{name}_trials"][f])
    np.testing.assert_allclose(x, d[f"{name}_x_9"], rtol=0, atol=1e-12 * np.abs(x).max())


@pytest.mark.parametrize("name", ["default", "aggressive"])
def test_oracle_chebyshev_matches_reference(name):
    """kind="chebyshev" (solvers.py:154-164, 306-311), incl. a non-descent fallback."""
    sc = scenes.c2(grid=(12, 3, 3), iterations=20)
    d = golden("frames_chebyshev.npz")
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                   factor="dense")
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(8):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=sc.iterations, m=sc.m, kind="chebyshev",
                                     rho=float(d[f"{name}_rho"]), S=int(d[f"{name}_S"]))
        q_prev, q_l = q_l, x
        np.testing.assert_allclose(rec.g, d[f"{name}_g"][f], rtol=1e-12)
        assert list(rec.ls_trials) == list(d[f"{name}_trials"][f])
        assert rec.fallbacks == int(d[f"{name}_fallbacks"][f])
    np.testing.assert_allclose(x, d[f"{name}_x_7"], rtol=0, atol=1e-12 * np.abs(x).max())


def test_oracle_lbfgs_scaled_identity_matches_reference():
    """lbfgs_init="scaled_identity" (solvers.py:136-141): no solve, r = rho/<t,t> q."""
    sc = scenes.c2(grid=(12, 3, 3), iterations=20)
    d = golden("frames_chebyshev.npz")
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                   factor="dense")
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(8):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=sc.iterations, m=sc.m,
                                     lbfgs_init="scaled_identity")
        q_prev, q_l = q_l, x
        np.testing.assert_allclose(rec.g, d["scaled_g"][f], rtol=1e-12)
        assert list(rec.ls_trials) == list(d["scaled_trials"][f])
    np.testing.assert_allclose(x, d["scaled_x_7"], rtol=0, atol=1e-12 * np.abs(x).max())


def test_oracle_cloth_hang_matches_reference_harness():
    """Spring networks (mass_spring, dynamics.py:111-151): cloth_hang.json."""
    from tests.helpers import ClothScene
    cs = ClothScene()
    d = golden("frames_cloth_hang.npz")
    assert np.array_equal(cs.fixed, d["fixed"])
    osys = O.build_springs(cs.verts, cs.edges, cs.rest, cs.faces, cs.density, cs.k, cs.h, cs.gravity, cs.fixed)
    q_l, q_prev = cs.q_l.copy(), cs.q_prev.copy()
    for f in range(int(d["frames"])):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=cs.iterations, m=cs.m)
        q_prev, q_l = q_l, x
        np.testing.assert_allclose(rec.g, d["g"][f], rtol=1e-12, atol=1e-18)
        assert list(rec.ls_trials) == list(d["trials"][f])
        if f"x_{f}" in d:
            np.testing.assert_allclose(x, d[f"x_{f}"], rtol=0, atol=1e-12 * np.abs(x).max())


@pytest.mark.parametrize("name", ["uniform", "two"])
def test_oracle_aniso_matches_reference(name):
    """Anisotropic fibres (dynamics.AnisoGroup, dynamics.py:154-193)."""
    from tests.helpers import aniso_cases
    sc = scenes.c1(grid=(10, 3, 3), iterations=10)
    d = golden("frames_aniso.npz")
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                   factor="dense", aniso=aniso_cases(sc.tets.shape[0])[name])
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(10):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=sc.iterations, m=sc.m)
        q_prev, q_l = q_l, x
        np.testing.assert_allclose(rec.g, d[f"{name}_g"][f], rtol=1e-12)
        assert list(rec.ls_trials) == list(d[f"{name}_trials"][f])
    np.testing.assert_allclose(x, d[f"{name}_x_9"], rtol=0, atol=1e-12 * np.abs(x).max())


def test_output_writers_match_reference_bytes(tmp_path):
    """CSV and OBJ output formats (harness.py:390-420, mesh.py:236-249) are
    byte-identical to the reference harness's files on the same records."""
    from paper_1604_07378_b200 import io as QIO
    from paper_1604_07378_b200.mesh import TetMesh
    from paper_1604_07378_b200.solvers import ConvergenceRecord
    d = golden("writers_inputs.npz")
    recs = [ConvergenceRecord(g=d[f"r{f}_g"].tolist(), ls_trials=d[f"r{f}_ls_trials"].tolist(),
                              cum_ms=d[f"r{f}_cum_ms"].tolist(), rel_error=d[f"r{f}_rel_error"].tolist())
            for f in range(2)]
    QIO.write_csv(str(tmp_path / "r.csv"), recs)
    assert (tmp_path / "r.csv").read_bytes() == open(os.path.join(os.path.dirname(FIX), "writers_report.csv"), "rb").read()
    sc = scenes.c1(grid=(4, 2, 2))
    QIO.export_frames([d["x0"]], str(tmp_path / "obj"), QIO.surface_triangles(TetMesh(sc.verts, sc.tets)))
    ref = open(os.path.join(os.path.dirname(FIX), "writers_obj", "frame_0000.obj"), "rb").read()
    assert (tmp_path / "obj" / "frame_0000.obj").read_bytes() == ref


def test_oracle_newton_matches_reference():
    """Newton frames (solvers.py:167-234) and newton_reference g* (:355-398).
    The central-difference Hessian divides rounding-level differences of the
    element gradient by the 1e-6 scale step, so frames agree to ~1e-11."""
    d = golden("frames_newton.npz")
    sc = scenes.c2(grid=(6, 2, 2), iterations=5)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                   factor="dense")
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(3):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=sc.iterations, kind="newton")
        q_prev, q_l = q_l, x
        np.testing.assert_allclose(rec.g, d["frames_g"][f], rtol=1e-9)
        assert list(rec.ls_trials) == list(d["frames_trials"][f])
    sc1 = scenes.c1()
    osys = O.build(sc1.verts, sc1.tets, sc1.density, oracle_material(sc1.material), sc1.h, sc1.gravity, sc1.fixed,
                   factor="dense")
    _, gs = O.newton_reference(osys, sc1.q_l.copy(), sc1.q_prev.copy())
    assert abs(gs - float(d["c1_gstar"])) <= 1e-12 * abs(gs)


def test_oracle_lbfgs_rest_pose_hessian_matches_reference():
    d = golden("frames_newton.npz")
    sc = scenes.c2(grid=(6, 2, 2), iterations=10)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                   factor="dense")
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for f in range(3):
        x, _, rec = O.simulate_frame(osys, q_l, q_prev, iterations=10, m=5, lbfgs_init="rest_pose_hessian")
        q_prev, q_l = q_l, x
        env = np.abs(d["rest_rev_g"][f] - d["rest_g"][f]).max() / np.abs(d["rest_g"][f]).max()
        assert np.abs(np.array(rec.g) - d["rest_g"][f]).max() / np.abs(d["rest_g"][f]).max() <= max(1e-10, 10 * env)
