"""Generate golden vectors from the UNMODIFIED reference (run in the build
container, where /root/reference exists; the GPU box never runs this).

    python tests/golden/make_golden.py [--quick] [--c4 | --colliders | --arap | --chebyshev | --cloth | --aniso | --writers | --newton (only those fixtures)]

Writes tests/golden/*.npz and copies the reference's own golden trajectories
(pkg/frontend/tests/fixtures/twist_{lbfgs,pd_qn}.csv) plus the bar_small asset
they were produced from into tests/golden/ref_fixtures/.  Inputs for the
configs come from paper_1604_07378_b200.scenes (seeded), fed to the reference
through its own Python API (build_system / SimState / simulate_frame), exactly
as SURVEY.md §8(d) prescribes.
"""

from __future__ import annotations

import os
import shutil
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, ROOT)

from qnsim import assets as ref_assets  # noqa: E402
from qnsim import dynamics as ref_dyn  # noqa: E402
from qnsim import linalg as ref_linalg  # noqa: E402
from qnsim import materials as ref_mat  # noqa: E402
from qnsim import mesh as ref_mesh  # noqa: E402
from qnsim import solvers as ref_solvers  # noqa: E402

from paper_1604_07378_b200 import scenes  # noqa: E402
from tests.helpers import aniso_cases, collider_bar_scene, material_specs  # noqa: E402


def ref_material(spec, name="custom"):
    def fn(s):
        if s[0] == "zero":
            return ref_mat.ZeroFn()
        if s[0] == "poly":
            return ref_mat.PolyFn(s[1])
        if s[0] == "log":
            return ref_mat.LogFn(s[1], s[2])
        return ref_mat.HermiteFn(s[1])
    return ref_mat.MaterialModel(a=fn(spec[0]), b=fn(spec[1]), c=fn(spec[2]), name=name)


MATERIAL_CASES = material_specs()


def gen_svd_materials():
    rng = np.random.default_rng(100)
    F = rng.standard_normal((1200, 3, 3))
    F[:100] = np.eye(3) + 1e-7 * rng.standard_normal((100, 3, 3))         # near rest (degenerate sigma)
    F[100:200] = F[100:200] * np.array([1.0, 1.0, -1.0])[None, :, None]   # reflections
    F[200:250, :, 2] = 0.0                                                 # exactly singular
    F[250:300] = 1e-12 * rng.standard_normal((50, 3, 3))                  # clamp region
    F[300] = np.eye(3)
    F[301] = np.diag([-1.0, 1.0, 1.0])
    F[302] = np.zeros((3, 3))
    U, s, V = ref_linalg.svd_rv_batch(F.copy())
    out = {"F": F, "sigma": s, "P_check": np.einsum("eab,eb,ecb->eac", U, s, V)}
    sig = np.concatenate([
        rng.uniform(0.2, 2.5, size=(400, 3)),
        np.column_stack([rng.uniform(0.5, 1.5, (100, 2)), -rng.uniform(0.001, 0.8, 100)]),  # inverted
        np.column_stack([rng.uniform(0.5, 1.5, (50, 2)), np.full(50, 1e-10)]),
        np.ones((1, 3)),
        rng.uniform(2.5, 4.0, size=(50, 3)),  # spline extrapolation
    ])
    out["mat_sigma"] = sig
    for name, spec in MATERIAL_CASES.items():
        mat = ref_material(spec, name)
        out[f"{name}_energy"] = ref_mat.vl_energy_batch(mat, sig)
        out[f"{name}_stress"] = ref_mat.vl_stress_batch(mat, sig)
        out[f"{name}_k"] = np.array(ref_mat.estimate_stiffness(mat))
        out[f"{name}_shift"] = np.array(mat.shift)
    np.savez_compressed(os.path.join(HERE, "svd_materials.npz"), **out)


def gen_meshes_elements():
    out = {}
    for key, (nx, ny, nz, size) in {"bar_c1": (20, 5, 5, (2.0, 0.5, 0.5)),
                                    "bar_small": (6, 2, 2, (0.6, 0.2, 0.2))}.items():
        v, t = ref_assets.bar_mesh(nx, ny, nz, size)
        out[f"{key}_verts"], out[f"{key}_tets"] = v, t
    sc = scenes.c1()
    mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=1000.0)
    G, vols = ref_mesh.tet_diff_operators(mesh)
    out["c1_masses"] = ref_mesh.lumped_masses(mesh)
    out["c1_vols"] = vols
    rng = np.random.default_rng(7)
    x = sc.verts + 0.02 * rng.standard_normal(sc.verts.shape)
    x[:30] = sc.verts[:30] * np.array([1.0, 1.0, -1.0]) + 0.3  # invert some tets
    out["c1_x"] = x
    for name, spec in MATERIAL_CASES.items():
        mat = ref_material(spec, name)
        k = ref_mat.estimate_stiffness(mat)
        grp = ref_dyn.VLGroup(sc.tets, G, vols, mat, k)
        out[f"c1_{name}_energy"] = np.array(grp.energy(x))
        g = np.zeros_like(x)
        grp.add_gradient(x, g)
        out[f"c1_{name}_grad"] = g
    np.savez_compressed(os.path.join(HERE, "meshes_elements.npz"), **out)


def run_reference(sc, mat_spec, frames, iterations, kind="lbfgs", save_frames=()):
    mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
    system = ref_dyn.build_system(mesh, ref_material(mat_spec), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    state = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    cfg = ref_solvers.SolverConfig(kind=kind, iterations=iterations, m=sc.m)
    g, tr, al, g0, pos = [], [], [], [], {}
    for f in range(frames):
        state, rec = ref_solvers.simulate_frame(system, state, cfg)
        g.append(rec.g)
        tr.append(rec.ls_trials)
        al.append(rec.alphas)
        g0.append(rec.g0)
        if f in save_frames:
            pos[f"x_{f}"] = state.q_l.copy()
    return dict(g=np.array(g), trials=np.array(tr), alphas=np.array(al), g0=np.array(g0), **pos)


def c4_spread_instances():
    """40 of the 1024 configs[3] instances: both ends of every 1/2/4/8-rank shard
    (shard_instances) plus evenly spread ones (>= 32 instances spread
    across ranks)."""
    ends = [r * 128 + o for r in range(8) for o in (0, 127)]
    spread = np.linspace(0, 1023, 24).round().astype(int).tolist()
    return sorted(set(ends + spread))


def gen_c4_spread(frames=10):
    t = time.time()
    sc4 = scenes.c4(instances=1024)
    keep = c4_spread_instances()
    out = {"instances": np.array(keep), "frames": frames}
    q_l, q_prev = sc4.q_l[0].copy(), sc4.q_prev[0].copy()
    for b in keep:
        sc4.q_l, sc4.q_prev = q_l, q_prev
        d = run_reference(sc4, sc4.batch_materials[b], frames, sc4.iterations, save_frames={frames - 1})
        for k, v in d.items():
            out[f"i{b}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "frames_c4_spread.npz"), **out)
    print("c4 spread", len(keep), "instances", time.time() - t)


def gen_frames(quick):
    t = time.time()
    sc = scenes.c1()
    fr = 20 if quick else 100
    d = run_reference(sc, sc.material, fr, sc.iterations, save_frames={0, 1, 9, 19, 49, 99})
    np.savez_compressed(os.path.join(HERE, "frames_c1_lbfgs.npz"), frames=fr, **d)
    d = run_reference(sc, sc.material, 10, sc.iterations, kind="pd_qn", save_frames={0, 9})
    np.savez_compressed(os.path.join(HERE, "frames_c1_pdqn.npz"), frames=10, **d)
    print("c1 frames", time.time() - t)
    # configs[3]: a few instances of the batch, first frames
    t = time.time()
    sc4 = scenes.c4(instances=1024)
    keep = [0, 1, 511, 1023]
    out = {"instances": np.array(keep)}
    for b in keep:
        sc4.q_l = sc4.q_l[0] if sc4.q_l.ndim == 3 else sc4.q_l
        sc4.q_prev = sc4.q_prev[0] if sc4.q_prev.ndim == 3 else sc4.q_prev
        d = run_reference(sc4, sc4.batch_materials[b], 3, sc4.iterations, save_frames={2})
        for k, v in d.items():
            out[f"i{b}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "frames_c4_subset.npz"), **out)
    print("c4 subset", time.time() - t)
    if not quick:  # configs[1] as-is (dense 15360^2 Cholesky): one frame, ~3 min
        t = time.time()
        sc2 = scenes.c2()
        d = run_reference(sc2, sc2.material, 1, sc2.iterations, save_frames={0})
        np.savez_compressed(os.path.join(HERE, "frames_c2_frame0.npz"), frames=1, **d)
        print("c2 frame 0", time.time() - t)


def ref_colliders(cols):
    out = []
    for c in cols:
        if c[0] == "halfspace":
            out.append(ref_dyn.HalfSpace(c[1], c[2]))
        elif c[0] == "sphere":
            out.append(ref_dyn.SphereCollider(c[1], c[2]))
        else:
            out.append(ref_dyn.TorusCollider(c[1], c[2], c[3]))
    return out


def gen_colliders():
    """Colliders: the reference's own sphere_drop scenario
    through its harness, and the three-collider bar through build_system."""
    from qnsim import harness as ref_harness
    t = time.time()
    scn = ref_harness.load_scenario(os.path.join(REF, "scenarios", "sphere_drop.json"))
    run = ref_harness.SimulationRun(scn)
    g, tr, al, g0, pos = [], [], [], [], {}
    frames = 30
    for f in range(frames):
        rec = run.step()
        g.append(rec.g)
        tr.append(rec.ls_trials)
        al.append(rec.alphas)
        g0.append(rec.g0)
        if f in (0, 9, 19, 29):
            pos[f"x_{f}"] = run.state.q_l.copy()
    # the same scenario with the tet list reversed (identical mathematics, another
    # summation order): penalty contact amplifies roundoff through active-set
    # flips, so this run is the reference's own roundoff envelope for parity
    mesh = run.system.mesh
    rmesh = ref_mesh.TetMesh(vertices=mesh.vertices.copy(), tets=mesh.tets[::-1].copy(), density=mesh.density)
    rsys = ref_dyn.build_system(rmesh, ref_harness._make_material(scn.material_spec), h=scn.h, gravity=scn.gravity,
                                fixed=[], colliders=scn.colliders, collision_weight=scn.collision_weight,
                                fit_interval=scn.fit_interval)
    rstate = ref_dyn.SimState(q_l=mesh.vertices.copy(), q_prev=mesh.vertices.copy())
    rg, rpos = [], {}
    for f in range(frames):
        rstate, rec = ref_solvers.simulate_frame(rsys, rstate, scn.solver)
        rg.append(rec.g)
        if f in (0, 9, 19, 29):
            rpos[f"rev_x_{f}"] = rstate.q_l.copy()
    np.savez_compressed(os.path.join(HERE, "frames_sphere_drop.npz"), frames=frames, g=np.array(g),
                        trials=np.array(tr), alphas=np.array(al), g0=np.array(g0), w_col=run.system.w_col,
                        rev_g=np.array(rg), **pos, **rpos)
    sc, cols = collider_bar_scene()
    mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
    system = ref_dyn.build_system(mesh, ref_material(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed,
                                  colliders=ref_colliders(cols))
    state = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    cfg = ref_solvers.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    g, tr, al, g0, pos, ncol = [], [], [], [], {}, []
    frames = 20
    for f in range(frames):
        state, rec = ref_solvers.simulate_frame(system, state, cfg)
        g.append(rec.g)
        tr.append(rec.ls_trials)
        al.append(rec.alphas)
        g0.append(rec.g0)
        ncol.append(ref_dyn.update_collisions(system, state, state.q_l).count)
        if f in (0, 4, 9, 19):
            pos[f"x_{f}"] = state.q_l.copy()
    np.savez_compressed(os.path.join(HERE, "frames_collider_bar.npz"), frames=frames, g=np.array(g),
                        trials=np.array(tr), alphas=np.array(al), g0=np.array(g0), w_col=system.w_col,
                        active=np.array(ncol), **pos)
    print("colliders", time.time() - t, "active per frame", ncol)


def gen_arap():
    """PD ARAP tets (PDMaterial("arap"), dynamics.ARAPGroup, SURVEY §8f row
    f3) through the reference's build_system: a bar of ARAP tets, and a bar
    whose tets alternate between ARAP and Neo-Hookean groups."""
    t = time.time()
    sc = scenes.c1(grid=(10, 3, 3), iterations=10)
    m = sc.tets.shape[0]
    out = {}
    half = np.arange(m) % 2 == 0
    cases = {"arap": ref_mat.PDMaterial(kind="arap", k=2e5),
             "mixed": [(np.nonzero(half)[0], ref_mat.PDMaterial(kind="arap", k=2e5)),
                       (np.nonzero(~half)[0], ref_material(sc.material))]}
    for name, mat in cases.items():
        mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
        system = ref_dyn.build_system(mesh, mat, h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
        state = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
        cfg = ref_solvers.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
        g, tr = [], []
        for f in range(10):
            state, rec = ref_solvers.simulate_frame(system, state, cfg)
            g.append(rec.g)
            tr.append(rec.ls_trials)
        out[f"{name}_g"], out[f"{name}_trials"], out[f"{name}_x_9"] = np.array(g), np.array(tr), state.q_l.copy()
    np.savez_compressed(os.path.join(HERE, "frames_arap.npz"), **out)
    print("arap", time.time() - t)


def gen_chebyshev():
    """Chebyshev-accelerated PD (solvers.py:154-164, 306-311) through the
    reference: the c2-like bar with seeded initial velocity, defaults
    (rho 0.9, S 10) and an aggressive (rho 0.99999, S 5) schedule that falls back once."""
    t = time.time()
    sc = scenes.c2(grid=(12, 3, 3), iterations=20)
    out = {}
    for name, rho, S in (("default", 0.9, 10), ("aggressive", 0.99999, 5)):
        mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
        system = ref_dyn.build_system(mesh, ref_material(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
        state = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
        cfg = ref_solvers.SolverConfig(kind="chebyshev", iterations=sc.iterations, rho=rho, S=S)
        g, tr, fb = [], [], []
        for f in range(8):
            state, rec = ref_solvers.simulate_frame(system, state, cfg)
            g.append(rec.g)
            tr.append(rec.ls_trials)
            fb.append(rec.fallbacks)
        out[f"{name}_g"], out[f"{name}_trials"] = np.array(g), np.array(tr)
        out[f"{name}_fallbacks"], out[f"{name}_x_7"] = np.array(fb), state.q_l.copy()
        out[f"{name}_rho"], out[f"{name}_S"] = rho, S
    # L-BFGS with the standard initial Hessian (lbfgs_init="scaled_identity", solvers.py:136-141)
    mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
    system = ref_dyn.build_system(mesh, ref_material(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    state = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    cfg = ref_solvers.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m, lbfgs_init="scaled_identity")
    g, tr = [], []
    for f in range(8):
        state, rec = ref_solvers.simulate_frame(system, state, cfg)
        g.append(rec.g)
        tr.append(rec.ls_trials)
    out["scaled_g"], out["scaled_trials"], out["scaled_x_7"] = np.array(g), np.array(tr), state.q_l.copy()
    # unconverged frames of this method carry roundoff into the next frame and
    # amplify it: the reference with its tet list reversed is the envelope
    rmesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets[::-1].copy(), density=sc.density)
    rsys = ref_dyn.build_system(rmesh, ref_material(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    rstate = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    rg = []
    for f in range(8):
        rstate, rec = ref_solvers.simulate_frame(rsys, rstate, cfg)
        rg.append(rec.g)
    out["scaled_rev_g"], out["scaled_rev_x_7"] = np.array(rg), rstate.q_l.copy()
    np.savez_compressed(os.path.join(HERE, "frames_chebyshev.npz"), **out)
    print("chebyshev", time.time() - t, {k: v for k, v in out.items() if k.endswith("fallbacks")})


def gen_cloth():
    """The reference's cloth_hang.json scenario (mass-spring network,
    SURVEY §8f row f3) through its harness."""
    from qnsim import harness as ref_harness
    t = time.time()
    scn = ref_harness.load_scenario(os.path.join(REF, "scenarios", "cloth_hang.json"))
    run = ref_harness.SimulationRun(scn)
    g, tr, pos = [], [], {}
    frames = 20
    for f in range(frames):
        rec = run.step()
        g.append(rec.g)
        tr.append(rec.ls_trials)
        if f in (0, 9, 19):
            pos[f"x_{f}"] = run.state.q_l.copy()
    np.savez_compressed(os.path.join(HERE, "frames_cloth_hang.npz"), frames=frames, g=np.array(g),
                        trials=np.array(tr), fixed=np.asarray(run.system.fixed), **pos)
    print("cloth", time.time() - t)


def gen_aniso():
    """Anisotropic fibres (dynamics.AnisoGroup) through the
    reference's build_system: every tet reinforced along one direction (the
    harness's "anisotropy" key), and two fibre families on alternating tets."""
    t = time.time()
    sc = scenes.c1(grid=(10, 3, 3), iterations=10)
    m = sc.tets.shape[0]
    cases = aniso_cases(m)
    out = {}
    for name, aniso in cases.items():
        mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
        system = ref_dyn.build_system(mesh, ref_material(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed,
                                      aniso=aniso)
        state = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
        cfg = ref_solvers.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
        g, tr = [], []
        for f in range(10):
            state, rec = ref_solvers.simulate_frame(system, state, cfg)
            g.append(rec.g)
            tr.append(rec.ls_trials)
        out[f"{name}_g"], out[f"{name}_trials"], out[f"{name}_x_9"] = np.array(g), np.array(tr), state.q_l.copy()
    np.savez_compressed(os.path.join(HERE, "frames_aniso.npz"), **out)
    print("aniso", time.time() - t)


def gen_writers():
    """The reference harness's output formats (harness.py:390-420): its
    write_csv on records of two reference frames, its surface_triangles and
    export_frames on the bar_small mesh."""
    from types import SimpleNamespace
    from qnsim import harness as ref_harness
    sc = scenes.c1(grid=(4, 2, 2), iterations=4)
    mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
    system = ref_dyn.build_system(mesh, ref_material(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    state = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    recs, states = [], []
    for _ in range(2):
        state, rec = ref_solvers.simulate_frame(system, state, ref_solvers.SolverConfig(kind="lbfgs", iterations=4))
        rec.cum_ms = [0.125 * (k + 1) for k in range(len(rec.g))]  # deterministic timing column
        rec.rel_error = [] if not recs else [1.0 / (k + 2) for k in range(len(rec.g))]
        recs.append(rec)
        states.append(state.q_l.copy())
    ref_harness.write_csv(os.path.join(HERE, "writers_report.csv"), SimpleNamespace(records=recs))
    d = os.path.join(HERE, "writers_obj")
    ref_harness.export_frames(states[:1], d, ref_mesh.surface_triangles(mesh))
    np.savez_compressed(os.path.join(HERE, "writers_inputs.npz"), x0=states[0],
                        **{f"r{f}_{k}": np.asarray(getattr(recs[f], k)) for f in range(2)
                           for k in ("g", "ls_trials", "cum_ms", "rel_error")})


def gen_newton():
    """Newton (solvers.py:167-234) frames and newton_reference g* (:355-398)
    through the reference: a 6x2x2 bar (3 frames x 5 Newton iterations) and
    the reference minimum of configs[0]'s first frame."""
    t = time.time()
    out = {}
    sc = scenes.c2(grid=(6, 2, 2), iterations=5)
    mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
    system = ref_dyn.build_system(mesh, ref_material(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    state = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    cfg = ref_solvers.SolverConfig(kind="newton", iterations=sc.iterations)
    g, tr = [], []
    for f in range(3):
        state, rec = ref_solvers.simulate_frame(system, state, cfg)
        g.append(rec.g)
        tr.append(rec.ls_trials)
    out["frames_g"], out["frames_trials"], out["frames_x_2"] = np.array(g), np.array(tr), state.q_l.copy()
    sc1 = scenes.c1()
    mesh = ref_mesh.TetMesh(vertices=sc1.verts, tets=sc1.tets, density=sc1.density)
    system = ref_dyn.build_system(mesh, ref_material(sc1.material), h=sc1.h, gravity=sc1.gravity, fixed=sc1.fixed)
    xs, gs = ref_solvers.newton_reference(system, ref_dyn.SimState(q_l=sc1.q_l.copy(), q_prev=sc1.q_prev.copy()))
    out["c1_gstar"], out["c1_xstar"] = gs, xs
    # L-BFGS with the rest-pose Hessian as the initial inverse (solvers.py:142-146, 401-407)
    mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
    system = ref_dyn.build_system(mesh, ref_material(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    state = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    cfg = ref_solvers.SolverConfig(kind="lbfgs", iterations=10, m=5, lbfgs_init="rest_pose_hessian")
    g, tr = [], []
    for f in range(3):
        state, rec = ref_solvers.simulate_frame(system, state, cfg)
        g.append(rec.g)
        tr.append(rec.ls_trials)
    out["rest_g"], out["rest_trials"], out["rest_x_2"] = np.array(g), np.array(tr), state.q_l.copy()
    # these frames converge to roundoff within the budget, so line-search
    # decisions at the noise floor (and the frame-end state) depend on the
    # summation order: the reference with its tet list reversed is the envelope
    rmesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets[::-1].copy(), density=sc.density)
    rsys = ref_dyn.build_system(rmesh, ref_material(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    rstate = ref_dyn.SimState(q_l=sc.q_l.copy(), q_prev=sc.q_prev.copy())
    rg = []
    for f in range(3):
        rstate, rec = ref_solvers.simulate_frame(rsys, rstate, cfg)
        rg.append(rec.g)
    out["rest_rev_g"], out["rest_rev_x_2"] = np.array(rg), rstate.q_l.copy()
    np.savez_compressed(os.path.join(HERE, "frames_newton.npz"), **out)
    print("newton", time.time() - t, gs)


def copy_fixtures():
    dst = os.path.join(HERE, "ref_fixtures")
    os.makedirs(dst, exist_ok=True)
    for src in ("frontend/tests/fixtures/twist_lbfgs.csv", "frontend/tests/fixtures/twist_pd_qn.csv",
                "assets/bar_small.node", "assets/bar_small.ele", "scenarios/bar_twist_small.json",
                "assets/sphere.node", "assets/sphere.ele", "scenarios/sphere_drop.json",
                "assets/cloth20.obj", "scenarios/cloth_hang.json"):
        shutil.copy(os.path.join(REF, src), os.path.join(dst, os.path.basename(src)))


if __name__ == "__main__":
    quick = "--quick" in sys.argv
    copy_fixtures()
    if "--c4" in sys.argv:
        gen_c4_spread()
        sys.exit(0)
    if "--colliders" in sys.argv:
        gen_colliders()
        sys.exit(0)
    if "--arap" in sys.argv:
        gen_arap()
        sys.exit(0)
    if "--chebyshev" in sys.argv:
        gen_chebyshev()
        sys.exit(0)
    if "--cloth" in sys.argv:
        gen_cloth()
        sys.exit(0)
    if "--aniso" in sys.argv:
        gen_aniso()
        sys.exit(0)
    if "--writers" in sys.argv:
        gen_writers()
        sys.exit(0)
    if "--newton" in sys.argv:
        gen_newton()
        sys.exit(0)
    gen_svd_materials()
    gen_meshes_elements()
    gen_frames(quick)
