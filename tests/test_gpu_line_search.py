"""Device line-search edge cases (run with -m gpu): the ascent -> SolverError
branch (solvers.py:244-246), StagnationError and the record padding
(solvers.py:250-252, 329-336), and non-default alpha_init / alpha_shrink.

The reference provokes ascent and stagnation by calling `line_search` with a
fabricated direction / gradient (pkg/tests/test_solvers.py:318-337).  The
device line search lives inside the frame graph, so the same situations are
injected there with the test-only `qn_system_set_fault` knob: mode 1 negates
the direction from iteration k on (slope > 0), mode 2 steps along -d while the
Armijo test keeps the slope of d (every trial raises g, the step underflows).
The first k-1 iterations are compared with the oracle's frame cut at k-1
iterations.
"""
import numpy as np
import pytest

import oracle.qnsim_oracle as O
import paper_1604_07378_b200 as Q
from paper_1604_07378_b200 import _lib, scenes
from paper_1604_07378_b200.materials import from_spec
from tests.helpers import oracle_material

pytestmark = pytest.mark.gpu

X_TOL = 1e-9
G_TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _gpu(built_lib):
    _lib.require_gpu()


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


@pytest.fixture(scope="module")
def c1():
    sc = scenes.c1(frames=1)
    mesh = Q.TetMesh(sc.verts, sc.tets, sc.density)
    system = Q.build_system(mesh, from_spec(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed,
                   factor="dense")
    yield sc, system, osys
    system.set_fault(0)


def state(sc):
    return Q.SimState(q_l=np.array(sc.q_l), q_prev=np.array(sc.q_prev))


@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("k", [1, 4])
def test_ascent_direction_raises_solver_error(c1, graph, k):
    sc, system, _ = c1
    system.set_graph_mode(graph)
    system.set_fault(1, k)
    try:
        with pytest.raises(Q.SolverError):
            Q.simulate_frame(system, state(sc), Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
    finally:
        system.set_fault(0)
        system.set_graph_mode(True)
    # the system is usable again afterwards and still matches the oracle
    st, rec = Q.simulate_frame(system, state(sc), Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
    x, _, ro = O.simulate_frame(c1[2], np.array(sc.q_l), np.array(sc.q_prev), iterations=sc.iterations, m=sc.m)
    assert rel(st.q_l, x) <= X_TOL and rel(rec.g, ro.g) <= G_TOL and not rec.stagnated


@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("kind", ["lbfgs", "pd_qn"])
@pytest.mark.parametrize("k", [1, 4])
def test_stagnation_pads_the_record(c1, graph, kind, k):
    """solvers.py:329-336: stagnated = True, the remaining iterations recorded as
    (g_x, 0 trials, alpha 0), positions = the last accepted iterate."""
    sc, system, osys = c1
    its = sc.iterations
    system.set_graph_mode(graph)
    system.set_fault(2, k)
    try:
        st, rec = Q.simulate_frame(system, state(sc), Q.SolverConfig(kind=kind, iterations=its, m=sc.m))
    finally:
        system.set_fault(0)
        system.set_graph_mode(True)
    assert rec.stagnated
    assert len(rec.g) == len(rec.ls_trials) == len(rec.alphas) == len(rec.cum_ms) == its
    if k > 1:
        x, y, ro = O.simulate_frame(osys, np.array(sc.q_l), np.array(sc.q_prev), iterations=k - 1, m=sc.m, kind=kind)
        assert not ro.stagnated
        assert rel(rec.g[:k - 1], ro.g) <= G_TOL
        assert rec.ls_trials[:k - 1] == ro.ls_trials
        np.testing.assert_array_equal(rec.alphas[:k - 1], ro.alphas)
        g_pad = ro.g[-1]
    else:
        x, y, ro = O.simulate_frame(osys, np.array(sc.q_l), np.array(sc.q_prev), iterations=1, m=sc.m, kind=kind,
                                    alpha_init=1e-13)  # stagnates at once in the oracle too
        assert ro.stagnated
        g_pad = ro.g0
    assert rel(rec.g[k - 1:], [g_pad] * (its - k + 1)) <= G_TOL
    assert rec.ls_trials[k - 1:] == [0] * (its - k + 1)
    assert rec.alphas[k - 1:] == [0.0] * (its - k + 1)
    assert rel(st.q_l, x) <= X_TOL


@pytest.mark.parametrize("alpha_init", [1e-12, 1.5e-12])
def test_alpha_floor_stagnation_without_injection(c1, alpha_init):
    """alpha_init * shrink below the 1e-12 floor: StagnationError before the first
    trial (solvers.py:250-252) in the reference and on the device; the frame
    returns y and a fully padded record."""
    sc, system, osys = c1
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m, alpha_init=alpha_init)
    st, rec = Q.simulate_frame(system, state(sc), cfg)
    x, _, ro = O.simulate_frame(osys, np.array(sc.q_l), np.array(sc.q_prev), iterations=sc.iterations, m=sc.m,
                                alpha_init=alpha_init)
    assert rec.stagnated and ro.stagnated
    assert rel(rec.g, ro.g) <= G_TOL and rec.ls_trials == ro.ls_trials == [0] * sc.iterations
    assert rel(st.q_l, x) <= X_TOL


@pytest.mark.parametrize("shrink", [0.9, 0.99])
def test_slow_shrink_reaches_stagnation_within_the_pass_bound(c1, shrink):
    """a line search with alpha_shrink close to 1 takes
    log(1e-12 / alpha_init) / log(shrink) trials (268 at 0.9, 2 750 at 0.99)
    before the floor; the device's runaway bound follows the configuration, so
    the frame ends stagnated like the reference instead of 'pass limit exceeded'."""
    sc, system, _ = c1
    system.set_fault(2, 2)
    try:
        st, rec = Q.simulate_frame(system, state(sc),
                                   Q.SolverConfig(kind="lbfgs", iterations=3, m=sc.m, alpha_shrink=shrink))
    finally:
        system.set_fault(0)
    assert rec.stagnated and rec.ls_trials[1:] == [0, 0]


def test_slow_shrink_parity_against_oracle(c1):
    """Non-default alpha_init / alpha_shrink without injection: identical trial
    counts and alphas, g and positions within the fp64 bar."""
    sc, system, osys = c1
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m, alpha_init=3.0, alpha_shrink=0.7,
                         gamma=0.45)
    st, rec = Q.simulate_frame(system, state(sc), cfg)
    x, _, ro = O.simulate_frame(osys, np.array(sc.q_l), np.array(sc.q_prev), iterations=sc.iterations, m=sc.m,
                                alpha_init=3.0, shrink=0.7, gamma=0.45)
    assert rec.ls_trials == ro.ls_trials
    np.testing.assert_array_equal(rec.alphas, ro.alphas)
    assert rel(rec.g, ro.g) <= G_TOL and rel(st.q_l, x) <= X_TOL


def test_shrink_at_least_one_is_refused(c1):
    sc, system, _ = c1
    with pytest.raises(Q.SolverError):
        Q.simulate_frame(system, state(sc), Q.SolverConfig(kind="lbfgs", iterations=2, alpha_shrink=1.0))


def test_fault_knob_arguments_checked(c1):
    _, system, _ = c1
    with pytest.raises(Exception):
        system.set_fault(3, 1)
    with pytest.raises(Exception):
        system.set_fault(1, 0)
    system.set_fault(0)


def test_pcg_stopping_at_maxit_is_reported():
    """a CG that stops at pcg_maxit short of pcg_tol raises instead of
    handing an inexact direction to the line search silently (device status
    bit 2 of the frame's error word; the host loop of the slab frame checks the
    same condition)."""
    sc = scenes.c5(grid=(12, 4, 4), frames=1)
    system = Q.build_system(Q.TetMesh(sc.verts, sc.tets, sc.density), from_spec(sc.material), h=sc.h,
                            gravity=sc.gravity, fixed=sc.fixed, solver="pcg", pcg_tol=1e-14, pcg_maxit=3)
    with pytest.raises(Q.SolverError, match="pcg_maxit"):
        Q.simulate_frame(system, state(sc), Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
    run = Q.ResidentRun(system, state(sc), Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
    with pytest.raises(Q.SolverError, match="pcg_maxit"):
        run.step()


def test_ascent_reported_by_the_resident_path(c1):
    """The device-resident step (no record requested) reports an ascent
    direction too, through the frame's error word."""
    sc, system, _ = c1
    system.set_fault(1, 2)
    try:
        run = Q.ResidentRun(system, state(sc), Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m))
        with pytest.raises(Q.SolverError):
            run.step()
    finally:
        system.set_fault(0)
