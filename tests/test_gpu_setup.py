"""Device setup assembly (csrc/qn_setup.cu) against the
numpy path (mesh.tet_diff_operators / lumped_masses, the reference's COO
assembly of L and A_free), run with -m gpu.  The device inverse is the
adjugate, so values agree to rounding (1e-13 relative), not bitwise; the
sparsity patterns are identical."""
import numpy as np
import pytest
import scipy.sparse

import oracle.qnsim_oracle as O
import paper_1604_07378_b200 as Q
from paper_1604_07378_b200 import _lib, scenes, setup
from paper_1604_07378_b200.materials import estimate_stiffness, from_spec
from paper_1604_07378_b200.mesh import VOLUME_EPS, TetMesh, lumped_masses, tet_diff_operators
from tests.helpers import oracle_material

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu(built_lib):
    _lib.require_gpu()


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


@pytest.mark.parametrize("name,grid", [("c5", (40, 10, 10)), ("c3", (30, 8, 8)), ("c1", (20, 5, 5))])
def test_device_assembly_matches_numpy(name, grid):
    sc = scenes.CONFIGS[name](grid=grid)
    mesh = TetMesh(sc.verts, sc.tets, sc.density)
    mat = from_spec(sc.material)
    k = estimate_stiffness(mat)
    G, vols, masses, L, Af = setup.assemble(sc.verts, sc.tets, sc.density, np.full(sc.tets.shape[0], k), sc.h,
                                            sc.fixed, VOLUME_EPS)
    G0, v0 = tet_diff_operators(mesh)
    m0 = lumped_masses(mesh)
    assert rel(G, G0) <= 1e-13 and rel(vols, v0) <= 1e-14 and rel(masses, m0) <= 1e-14
    w = v0 * k
    GG = np.einsum("evc,euc->evu", G0, G0)
    n = mesh.n
    L0 = scipy.sparse.coo_matrix(((w[:, None, None] * GG).reshape(-1),
                                  (np.repeat(sc.tets, 4, axis=1).reshape(-1), np.tile(sc.tets, (1, 4)).reshape(-1))),
                                 shape=(n, n)).tocsr()
    L0.sort_indices()
    assert np.array_equal(L.indptr, L0.indptr) and np.array_equal(L.indices, L0.indices)
    assert rel(L.data, L0.data) <= 1e-12
    mask = np.ones(n, bool)
    mask[sc.fixed] = False
    free = np.nonzero(mask)[0]
    A0 = (L0 + scipy.sparse.diags(m0 / sc.h ** 2)).tocsr()[free][:, free].tocsr()
    A0.sort_indices()
    assert np.array_equal(Af.indptr, A0.indptr) and np.array_equal(Af.indices, A0.indices)
    assert rel(Af.data, A0.data) <= 1e-12


def test_device_setup_frames_against_oracle(monkeypatch):
    """build_system on the device-assembled system (forced below the size
    threshold) gives the oracle's frames at the north_star bar."""
    monkeypatch.setenv("QN_DEVICE_SETUP", "1")
    sc = scenes.c5(grid=(40, 10, 10), frames=2)
    system = Q.build_system(Q.TetMesh(sc.verts, sc.tets, sc.density), from_spec(sc.material), h=sc.h,
                            gravity=sc.gravity, fixed=sc.fixed, solver="amg", pcg_tol=1e-10)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    st = Q.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    q_l, q_prev = sc.q_l.copy(), sc.q_prev.copy()
    for _ in range(2):
        st, rec = Q.simulate_frame(system, st, cfg)
        x, _, ro = O.simulate_frame(osys, q_l, q_prev, iterations=sc.iterations, m=sc.m)
        q_prev, q_l = q_l, x
        assert rel(st.q_l, x) <= 1e-9 and rel(rec.g, ro.g) <= 1e-10 and rec.ls_trials == ro.ls_trials


def test_device_setup_direct_solver_and_two_groups(monkeypatch):
    """Group-major tet order (two materials) and the direct factor on the
    device-assembled A_free."""
    monkeypatch.setenv("QN_DEVICE_SETUP", "1")
    sc = scenes.c1(frames=1)
    half = sc.tets.shape[0] // 2
    idx_a, idx_b = np.arange(half, sc.tets.shape[0]), np.arange(half)
    mats = [(idx_a, Q.make_builtin("neohookean", {"mu": 2e5, "lambda": 5e5})),
            (idx_b, Q.make_builtin("stvk", {"mu": 1e5, "lambda": 3e5}))]
    mesh = Q.TetMesh(sc.verts, sc.tets, sc.density)
    a = Q.build_system(mesh, mats, h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    monkeypatch.setenv("QN_DEVICE_SETUP", "0")
    b = Q.build_system(mesh, mats, h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    assert rel(a.L.toarray(), b.L.toarray()) <= 1e-12
    cfg = Q.SolverConfig(kind="lbfgs", iterations=10, m=5)
    sa, ra = Q.simulate_frame(a, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev), cfg)
    sb, rb = Q.simulate_frame(b, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev), cfg)
    assert rel(sa.q_l, sb.q_l) <= 1e-12 and rel(ra.g, rb.g) <= 1e-12


def test_device_setup_rejects_degenerate_tets():
    verts = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 0]])
    tets = np.array([[0, 1, 2, 3], [0, 1, 4, 2]])  # second tet is flat (all in z = 0)
    with pytest.raises(ValueError, match="degenerate"):
        setup.assemble(verts, tets, 1000.0, np.ones(2), 1 / 30, [], VOLUME_EPS)
    with pytest.raises(ValueError):
        setup.assemble(verts, np.array([[0, 1, 2, 7]]), 1000.0, np.ones(1), 1 / 30, [], VOLUME_EPS)
