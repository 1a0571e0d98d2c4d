"""Seeded synthetic inputs for the BASELINE.json configs (c1..c5).

Plain numpy arrays only (no GPU, no oracle): the same host arrays feed the B200
path and the CPU oracle.  The reference cannot express these scenes through
its scenario JSON (SURVEY.md §5 "Config and flags"), so they are built here
through the API, exactly as SURVEY.md §8(d) prescribes:

* mesh: `bar_mesh(nx, ny, nz, size=(0.1 nx, 0.1 ny, 0.1 nz))` (Freudenthal
  6-tet split, reference `assets.py:10-69`, vectorised in `mesh.grid_bar`) with
  U(-0.001, 0.001) m jitter per coordinate from `default_rng(seed)`;
* density 1000, h = 1/30, gravity (0, 0, -9.81);
* pinned vertices chosen by GRID INDEX (the i = 0 plane, plus i = nx for c3),
  not by a coordinate box, because the jitter moves the face off x = 0;
* mu = E / (2 (1 + nu)), lambda = E nu / ((1 + nu)(1 - 2 nu)).

Material specs are generic Valanis-Landel triples: each of a, b, c is one of
("zero",), ("poly", coeffs_ascending), ("log", alpha, beta), ("hermite", knots[K,3]).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_1604_07378_b200.mesh import grid_bar

H = 1.0 / 30.0
GRAVITY = (0.0, 0.0, -9.81)
DENSITY = 1000.0
SPACING = 0.1
JITTER = 0.001


def lame(E, nu):
    return E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))


def builtin_spec(name, mu=None, lam=0.0, mu1=None, mu2=0.0):
    """Generic (a, b, c) spec of the reference built-ins (materials.py:257-289)."""
    if name == "neohookean":
        return (("poly", [-mu / 2.0, 0.0, mu / 2.0]), ("zero",), ("log", -mu, lam))
    if name == "stvk":
        A = mu / 4.0 + lam / 8.0
        return (("poly", [A + lam / 2.0, 0.0, -2 * A - lam / 2.0, 0.0, A]),
                ("poly", [-lam / 4.0, 0.0, lam / 4.0]), ("zero",))
    if name == "polynomial":
        return (("poly", list(mu * np.array([1, -4, 6, -4, 1.0]))), ("zero",), ("zero",))
    if name == "corotated":
        return (("poly", [mu + 1.5 * lam, -2 * mu - 3 * lam, mu + 0.5 * lam]), ("poly", [0.0, lam]), ("zero",))
    if name == "mooney_rivlin":
        b = ("poly", [-mu2, 0.0, mu2]) if mu2 > 0 else ("zero",)
        return (("poly", [-mu1, 0.0, mu1]), b, ("log", -(2 * mu1 + 4 * mu2), lam))
    raise ValueError(f"unknown builtin {name!r}")


@dataclass
class Scene:
    name: str
    verts: np.ndarray            # (n, 3) rest positions
    tets: np.ndarray             # (m, 4)
    fixed: np.ndarray            # sorted vertex ids
    material: tuple              # generic spec (single system)
    q_l: np.ndarray              # (n, 3) or (B, n, 3) for batches
    q_prev: np.ndarray
    iterations: int
    frames: int
    m: int = 5
    h: float = H
    gravity: tuple = GRAVITY
    density: float = DENSITY
    batch_materials: list = field(default_factory=list)  # per-instance specs (c4)
    grid: tuple = ()

    @property
    def batch(self):
        return len(self.batch_materials)


def jittered_bar(nx, ny, nz, rng):
    verts, tets = grid_bar(nx, ny, nz, (SPACING * nx, SPACING * ny, SPACING * nz))
    verts = verts + rng.uniform(-JITTER, JITTER, size=verts.shape)
    return verts, tets


def face_ids(nx, ny, nz, i):
    """Vertex ids of grid plane i (vid = (i(ny+1)+j)(nz+1)+k, assets.py:25-26)."""
    per = (ny + 1) * (nz + 1)
    return np.arange(i * per, (i + 1) * per, dtype=np.int64)


def c1(seed=0, frames=100, iterations=10, grid=(20, 5, 5)):
    """configs[0]: cantilever NH, E=5e5, nu=0.45, 20x5x5, 100 frames x 10 its."""
    rng = np.random.default_rng(seed)
    verts, tets = jittered_bar(*grid, rng)
    mu, lam = lame(5e5, 0.45)
    q = verts.copy()
    return Scene("c1_cantilever_nh", verts, tets, face_ids(*grid, 0), builtin_spec("neohookean", mu, lam),
                 q, q.copy(), iterations, frames, grid=grid)


def c2(seed=1, frames=50, iterations=20, grid=(60, 15, 15)):
    """configs[1]: cantilever StVK, E=1e6, nu=0.4, 60x15x15, v0 ~ N(0, 0.05^2), 50 frames x 20 its."""
    rng = np.random.default_rng(seed)
    verts, tets = jittered_bar(*grid, rng)
    mu, lam = lame(1e6, 0.4)
    fixed = face_ids(*grid, 0)
    v0 = rng.normal(0.0, 0.05, size=verts.shape)
    v0[fixed] = 0.0
    q = verts.copy()
    return Scene("c2_cantilever_stvk", verts, tets, fixed, builtin_spec("stvk", mu, lam),
                 q, q - H * v0, iterations, frames, grid=grid)


def nh_spline_spec(rng, E=5e5, nu=0.45, knots=8, lo=0.3, hi=3.0):
    """Hermite splines through Neo-Hookean a and c values (b = 0) at `knots`
    stretches in [lo, hi], values and tangents scaled per knot by U(0.8, 1.5)."""
    mu, lam = lame(E, nu)
    xs = np.linspace(lo, hi, knots)
    sa = rng.uniform(0.8, 1.5, size=knots)
    sc = rng.uniform(0.8, 1.5, size=knots)
    a_pts = np.stack([xs, sa * (0.5 * mu * (xs * xs - 1.0)), sa * (mu * xs)], axis=1)
    lx = np.log(xs)
    c_pts = np.stack([xs, sc * (-mu * lx + 0.5 * lam * lx * lx), sc * ((-mu + lam * lx) / xs)], axis=1)
    return (("hermite", a_pts), ("zero",), ("hermite", c_pts))


def twisted(verts, fixed_mask, lx, amplitude):
    """Rotation of each cross-section about the bar axis by theta(x) =
    theta_max sin(pi x / lx); theta_max makes the middle cross-section's
    outermost vertex move `amplitude` m (chord).  Pinned vertices stay put."""
    cy = 0.5 * (verts[:, 1].max() + verts[:, 1].min())
    cz = 0.5 * (verts[:, 2].max() + verts[:, 2].min())
    r = np.hypot(verts[:, 1] - cy, verts[:, 2] - cz)
    theta_max = 2.0 * np.arcsin(min(1.0, amplitude / (2.0 * r.max())))
    th = theta_max * np.sin(np.pi * np.clip(verts[:, 0] / lx, 0.0, 1.0))
    c, s = np.cos(th), np.sin(th)
    q = verts.copy()
    dy, dz = verts[:, 1] - cy, verts[:, 2] - cz
    q[:, 1] = cy + c * dy - s * dz
    q[:, 2] = cz + s * dy + c * dz
    q[fixed_mask] = verts[fixed_mask]
    return q


def c3(seed=2, frames=30, iterations=10, grid=(100, 25, 25), twist=0.2):
    """configs[2]: spline VL bar, both ends pinned, 0.2 m initial twist."""
    rng = np.random.default_rng(seed)
    verts, tets = jittered_bar(*grid, rng)
    fixed = np.concatenate([face_ids(*grid, 0), face_ids(*grid, grid[0])])
    mask = np.zeros(verts.shape[0], dtype=bool)
    mask[fixed] = True
    q = twisted(verts, mask, SPACING * grid[0], twist)
    return Scene("c3_spline_twist", verts, tets, fixed, nh_spline_spec(rng), q, q.copy(), iterations,
                 frames, grid=grid)


def c4(seed=3, instances=1024, frames=60, iterations=10, grid=(20, 5, 5)):
    """configs[3]: `instances` copies of the c1 mesh, NH with per-instance
    E ~ U(1e5, 1e6), nu ~ U(0.3, 0.48)."""
    base = c1(seed=0, grid=grid)
    rng = np.random.default_rng(seed)
    E = rng.uniform(1e5, 1e6, size=instances)
    nu = rng.uniform(0.3, 0.48, size=instances)
    mats = [builtin_spec("neohookean", *lame(e, v)) for e, v in zip(E, nu)]
    q = np.broadcast_to(base.verts, (instances,) + base.verts.shape).copy()
    return Scene("c4_batch_nh", base.verts, base.tets, base.fixed, mats[0], q, q.copy(), iterations, frames,
                 batch_materials=mats, grid=grid)


def c5(seed=4, frames=5, iterations=10, grid=(400, 100, 100)):
    """configs[4]: large polynomial bar: Neo-Hookean plus a seeded cubic term
    c3 (x^2 - 1)^3 in a(x) (separable restatement of "cubic in (I1 - 3)",
    SURVEY.md §8d), E = 5e5, nu = 0.45, c3 = mu U(0.05, 0.2)."""
    rng = np.random.default_rng(seed)
    verts, tets = jittered_bar(*grid, rng)
    spec = _c5_material(rng)
    q = verts.copy()
    return Scene("c5_large_poly", verts, tets, face_ids(*grid, 0), spec, q, q.copy(), iterations, frames,
                 grid=grid)


def c5_vertices(seed=4, grid=(400, 100, 100)):
    """configs[4] without the global tet array (each slab generates its own
    cells with mesh.grid_bar_cells): jittered rest vertices, material spec and
    pinned ids, drawn from the same seeded stream as c5()."""
    from paper_1604_07378_b200.mesh import grid_bar_verts
    rng = np.random.default_rng(seed)
    nx, ny, nz = grid
    verts = grid_bar_verts(nx, ny, nz, (SPACING * nx, SPACING * ny, SPACING * nz))
    verts = verts + rng.uniform(-JITTER, JITTER, size=verts.shape)
    return verts, _c5_material(rng), face_ids(*grid, 0)


def _c5_material(rng):
    mu, lam = lame(5e5, 0.45)
    k3 = mu * rng.uniform(0.05, 0.2)
    a = np.array([-mu / 2.0, 0.0, mu / 2.0, 0.0, 0.0, 0.0, 0.0])
    a = a + k3 * np.array([-1.0, 0.0, 3.0, 0.0, -3.0, 0.0, 1.0])
    return (("poly", list(a)), ("zero",), ("log", -mu, lam))


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
