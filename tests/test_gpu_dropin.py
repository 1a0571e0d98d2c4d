"""The drop-in, exercised inside the reference's own code (run with -m gpu).

INTEGRATION.md §1 swaps `qnsim.harness.build_system / simulate_frame /
newton_reference` (imported into the harness namespace, harness.py:27-34) for
this package's and drives the UNMODIFIED `harness.SimulationRun.step`
(harness.py:346-351) on the reference's bar_twist_small scenario; §2 keeps the
reference's whole `simulate_frame` loop (solvers.py:260-352) and plugs the B200
`sysfact` (linalg.Factorization duck type, solvers.py:116,134) and element
groups (VLGroup duck type, dynamics.py:464-465,473-474) into a reference
`SimSystem`.

The reference package is the one installed (unmodified, `pip install --target
baseline/_ref`) into baseline/_ref, which travels to the GPU box
with the repo snapshot; the tests skip when it is absent.
"""
import copy
import json
import os
import sys

import numpy as np
import pytest

import paper_1604_07378_b200 as Q
from paper_1604_07378_b200 import _lib, scenes
from tests.helpers import FIX, read_csv

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SITE = os.path.join(ROOT, "baseline", "_ref")
X_TOL = 1e-9
G_TOL = 1e-10


@pytest.fixture(scope="module")
def qnsim():
    if not os.path.isdir(os.path.join(REF_SITE, "qnsim")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF_SITE)
    try:
        import qnsim as ref
        import qnsim.harness  # noqa: F401
    finally:
        sys.path.remove(REF_SITE)
    _lib.require_gpu()
    return ref


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def twist_scenario(ref, frames):
    with open(os.path.join(FIX, "bar_twist_small.json")) as fh:
        raw = json.load(fh)
    raw["mesh"]["node"], raw["mesh"]["ele"] = "bar_small.node", "bar_small.ele"
    raw["frames"] = frames
    raw["solver"]["iterations"] = 20
    return ref.harness.parse_scenario(raw, base_dir=FIX)


@pytest.fixture
def swapped_harness(qnsim):
    h = qnsim.harness
    saved = (h.build_system, h.simulate_frame, h.newton_reference)
    h.build_system, h.simulate_frame, h.newton_reference = Q.build_system, Q.simulate_frame, Q.newton_reference
    yield h
    h.build_system, h.simulate_frame, h.newton_reference = saved


@pytest.mark.parametrize("kind", ["lbfgs", "pd_qn"])
def test_harness_simulation_run_with_the_b200_frame(qnsim, swapped_harness, kind):
    """§1: the reference harness, its scenario parser, fixed-group motion and
    SimulationRun.step, with the B200 build_system / simulate_frame in its
    namespace, reproduces the reference's own golden CSVs (twist_{kind}.csv)."""
    g_ref, tr_ref = read_csv(os.path.join(FIX, f"twist_{kind}.csv"))
    scn = twist_scenario(qnsim, g_ref.shape[0])
    scn.solver = qnsim.SolverConfig(kind=kind, iterations=20, m=5)
    sim = swapped_harness.SimulationRun(scn)
    assert isinstance(sim.system, Q.SimSystem)  # the harness built the device system
    for f in range(g_ref.shape[0]):
        rec = sim.step()
        assert rel(rec.g, g_ref[f]) <= G_TOL, f
        assert list(rec.ls_trials) == list(tr_ref[f]), f


def test_harness_run_writes_the_reference_csv_schema(qnsim, swapped_harness, tmp_path):
    """harness.run (harness.py:354-388): records, relative errors from the B200
    newton_reference on the recorded frames, and the CSV writer."""
    scn = twist_scenario(qnsim, 3)
    scn.solver = qnsim.SolverConfig(kind="lbfgs", iterations=20, m=5)
    scn.outputs = {"record_frames": [2], "csv": str(tmp_path / "out.csv")}
    rep = swapped_harness.run(scn, out_dir=str(tmp_path))
    g_ref, tr_ref = read_csv(os.path.join(FIX, "twist_lbfgs.csv"))
    for f, rec in enumerate(rep.records):
        assert rel(rec.g, g_ref[f]) <= G_TOL
    assert 2 in rep.final_rel_errors and np.isfinite(rep.final_rel_errors[2])
    with open(tmp_path / "out.csv") as fh:
        assert fh.readline().strip() == swapped_harness.CSV_HEADER


def _ref_material(ref, spec):
    def fn(s):
        return {"zero": lambda: ref.materials.ZeroFn(), "poly": lambda: ref.materials.PolyFn(s[1]),
                "log": lambda: ref.materials.LogFn(s[1], s[2]), "hermite": lambda: ref.materials.HermiteFn(s[1])}[s[0]]()
    return ref.materials.MaterialModel(a=fn(spec[0]), b=fn(spec[1]), c=fn(spec[2]), name="custom")


@pytest.mark.parametrize("name", ["c1", "c3_small"])
def test_seams_inside_the_unmodified_reference_loop(qnsim, name):
    """§2: reference simulate_frame with the B200 sysfact and element groups vs
    the same loop with the reference's own (dense Cholesky, numpy VLGroup)."""
    sc = scenes.c1(frames=3) if name == "c1" else scenes.c3(grid=(12, 4, 4), frames=3)
    ref = qnsim
    mesh = ref.mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
    mat = _ref_material(ref, sc.material)
    sys_ref = ref.build_system(mesh, mat, h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    sys_gpu = Q.build_system(mesh, mat, h=sc.h, gravity=sc.gravity, fixed=sc.fixed)  # reference objects adopted
    sys_mix = copy.copy(sys_ref)
    sys_mix.sysfact = sys_gpu.sysfact
    sys_mix.groups = sys_gpu.groups
    cfg = ref.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    st_a = ref.SimState(q_l=np.array(sc.q_l), q_prev=np.array(sc.q_prev))
    st_b = ref.SimState(q_l=np.array(sc.q_l), q_prev=np.array(sc.q_prev))
    for f in range(3):
        st_a, ra = ref.simulate_frame(sys_ref, st_a, cfg)
        st_b, rb = ref.simulate_frame(sys_mix, st_b, cfg)
        assert rel(rb.g, ra.g) <= G_TOL, f
        assert rb.ls_trials == ra.ls_trials, f
        assert rel(st_b.q_l, st_a.q_l) <= X_TOL, f


def test_reference_objects_are_adopted(qnsim):
    """build_system accepts qnsim's TetMesh / MaterialModel / FitInterval /
    colliders (paper_1604_07378_b200.adopt) and gives the same system as this
    package's own types."""
    ref = qnsim
    sc = scenes.c1(frames=1)
    mat = ref.materials.make_builtin("neohookean", {"mu": 1e5, "lambda": 4e5})
    mesh = ref.mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
    col = [ref.dynamics.HalfSpace((0, 0, -0.05), (0, 0, 1))]
    a = Q.build_system(mesh, mat, h=sc.h, gravity=sc.gravity, fixed=sc.fixed, colliders=col,
                       fit_interval=ref.materials.FitInterval())
    b = Q.build_system(Q.TetMesh(sc.verts, sc.tets, sc.density), Q.make_builtin("neohookean", {"mu": 1e5, "lambda": 4e5}),
                       h=sc.h, gravity=sc.gravity, fixed=sc.fixed, colliders=[Q.dynamics.HalfSpace((0, 0, -0.05), (0, 0, 1))])
    cfg = Q.SolverConfig(kind="lbfgs", iterations=10, m=5)
    sa, ra = Q.simulate_frame(a, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev), cfg)
    sb, rb = Q.simulate_frame(b, Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev), cfg)
    np.testing.assert_array_equal(sa.q_l, sb.q_l)
    assert ra.g == rb.g
