"""numpy/scipy restatement of the qnsim hot path (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Reference = `/root/reference/pkg/src/qnsim` (pure Python, numpy + scipy).  The
restatement keeps the reference's arithmetic (same library primitives, same
operation order where it matters) so it agrees with the reference to roundoff;
`tests/test_oracle_golden.py` pins it to the reference's own outputs.

Differences from the reference, all deliberate and documented in DESIGN.md:
* the prefactored solve can use a sparse LU (`factor="sparse"`) in place of the
  dense `cho_factor` of `linalg.py:31` / `dynamics.py:413` (dense is O(n^2)
  memory, infeasible beyond configs[1]); `factor="dense"` restates the
  reference exactly; for configs[4] (12 M dofs, sparse LU infeasible too)
  `factor="cg"` solves with Jacobi-PCG to 1e-13 (oracle/cg_free.c);
* the harness-side scenario parsing, PD materials, Chebyshev and Newton are
  out of the hot-path scope and not restated; colliders
  (§8f row f2) are restated below.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

SIGMA_CLAMP = 1e-10          # linalg.py:13
LOG_EPS = 0.01               # materials.py:21
FIT_SAMPLES = 1001           # materials.py:23
CURVATURE_GUARD = 1e-12      # solvers.py:28
ALPHA_FLOOR = 1e-12          # solvers.py:29


class OracleError(Exception):
    pass


class OracleStagnation(OracleError):
    pass


# --------------------------------------------------------------------------
# mesh (setup)

_FREUDENTHAL = np.array(
    [(0, 1, 3, 7), (0, 3, 2, 7), (0, 2, 6, 7), (0, 6, 4, 7), (0, 4, 5, 7), (0, 5, 1, 7)],
    dtype=np.int64,
)  # assets.py:10-17 (corner code = di*4 + dj*2 + dk)


def grid_bar(nx, ny, nz, size):
    """Vectorised restatement of `assets.bar_mesh` (assets.py:20-69, 66-69).

    Vertex id (i*(ny+1)+j)*(nz+1)+k (assets.py:25-26), cells in C order, six
    tets per cell in `_CUBE_TETS` order, then the orientation fix that swaps
    corners 2,3 of negatively oriented tets (assets.py:58-62)."""
    sx, sy, sz = size[0] / nx, size[1] / ny, size[2] / nz
    i, j, k = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    verts = np.stack([0.0 + i.ravel() * sx, 0.0 + j.ravel() * sy, 0.0 + k.ravel() * sz], axis=1)
    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    corners = np.empty((ci.size, 8), dtype=np.int64)
    for code in range(8):
        di, dj, dk = code >> 2, (code >> 1) & 1, code & 1
        corners[:, code] = ((ci + di) * (ny + 1) + (cj + dj)) * (nz + 1) + (ck + dk)
    tets = corners[:, _FREUDENTHAL].reshape(-1, 4)
    v = verts[tets]
    vols = np.linalg.det(np.swapaxes(v[:, 1:] - v[:, :1], 1, 2)) / 6.0
    neg = vols < 0
    tets[neg] = tets[neg][:, [0, 1, 3, 2]]
    return verts, tets


def read_node_ele(node_path, ele_path):
    """TetGen reader restating mesh.py:52-68,71-146 for well-formed files
    (comments stripped, 0/1-based detection, orientation fix)."""
    def rows(path):
        out = []
        with open(path) as fh:
            for line in fh:
                t = line.split("#", 1)[0].strip()
                if t:
                    out.append(t.split())
        return out

    nr = rows(node_path)
    nv = int(nr[0][0])
    ids = np.array([int(r[0]) for r in nr[1:1 + nv]])
    verts = np.array([[float(r[1]), float(r[2]), float(r[3])] for r in nr[1:1 + nv]])
    base = 0 if ids[0] == 0 else 1
    er = rows(ele_path)
    ne = int(er[0][0])
    tets = np.array([[int(p) for p in r[1:5]] for r in er[1:1 + ne]], dtype=np.int64) - base
    v = verts[tets]
    vols = np.linalg.det(v[:, 1:] - v[:, :1]) / 6.0
    neg = vols < 0
    tets[neg] = tets[neg][:, [0, 1, 3, 2]]
    return verts, tets


def diff_operators(verts, tets):
    """G (m,4,3) with G[1:] = Dm^-1, G[0] = -sum rows; volumes (mesh.py:200-216)."""
    v = verts[tets]
    Dm = np.swapaxes(v[:, 1:] - v[:, :1], 1, 2)
    vols = np.linalg.det(Dm) / 6.0
    if np.any(vols < 1e-14):
        raise OracleError("degenerate rest tet")
    Dinv = np.linalg.inv(Dm)
    G = np.empty((tets.shape[0], 4, 3))
    G[:, 1:, :] = Dinv
    G[:, 0, :] = -Dinv.sum(axis=1)
    return G, vols


def vertex_masses(verts, tets, density):
    """Lumped masses rho*V/4 per corner, corner-major accumulation (mesh.py:178-197)."""
    v = verts[tets]
    vols = np.linalg.det(v[:, 1:] - v[:, :1]) / 6.0
    share = density * vols / 4.0
    m = np.zeros(verts.shape[0])
    for c in range(4):
        np.add.at(m, tets[:, c], share)
    if np.any(m <= 0):
        raise OracleError("massless vertex")
    return m


# --------------------------------------------------------------------------
# scalar functions and Valanis-Landel materials (materials.py)

class Zero:
    """materials.py:32-37"""
    kind = "zero"

    def f(self, x):
        return np.zeros_like(np.asarray(x, dtype=np.float64))

    df = f


class Poly:
    """Ascending coefficients, numpy polyval (Horner) — materials.py:40-51."""
    kind = "poly"

    def __init__(self, coeffs):
        self.c = np.asarray(coeffs, dtype=np.float64)
        self.dc = np.polynomial.polynomial.polyder(self.c) if self.c.size > 1 else np.zeros(1)

    def f(self, x):
        return np.polynomial.polynomial.polyval(np.asarray(x, dtype=np.float64), self.c)

    def df(self, x):
        return np.polynomial.polynomial.polyval(np.asarray(x, dtype=np.float64), self.dc)


class Log:
    """alpha ln x + beta/2 ln^2 x, quadratic Taylor continuation at x <= eps (materials.py:54-80)."""
    kind = "log"

    def __init__(self, alpha, beta, eps=LOG_EPS):
        self.alpha, self.beta, self.eps = float(alpha), float(beta), float(eps)
        le = np.log(self.eps)
        self.f0 = self.alpha * le + 0.5 * self.beta * le * le
        self.f1 = (self.alpha + self.beta * le) / self.eps
        self.f2 = (self.beta - self.alpha - self.beta * le) / (self.eps * self.eps)

    def f(self, x):
        x = np.asarray(x, dtype=np.float64)
        inside = x > self.eps
        lx = np.log(np.where(inside, x, 1.0))
        d = x - self.eps
        return np.where(inside, self.alpha * lx + 0.5 * self.beta * lx * lx,
                        self.f0 + self.f1 * d + 0.5 * self.f2 * d * d)

    def df(self, x):
        x = np.asarray(x, dtype=np.float64)
        inside = x > self.eps
        sx = np.where(inside, x, 1.0)
        return np.where(inside, (self.alpha + self.beta * np.log(sx)) / sx,
                        self.f1 + self.f2 * (x - self.eps))


class Hermite:
    """Cubic Hermite spline, searchsorted(side='right') segments clipped to the
    knot range, linear extrapolation outside (materials.py:83-133)."""
    kind = "hermite"

    def __init__(self, points):
        p = np.asarray(points, dtype=np.float64)
        p = p[np.argsort(p[:, 0])]
        if p.shape[0] < 2 or np.any(np.diff(p[:, 0]) <= 0):
            raise OracleError("bad spline knots")
        self.xs, self.ys, self.ts = p[:, 0].copy(), p[:, 1].copy(), p[:, 2].copy()

    def _seg(self, x):
        i = np.clip(np.searchsorted(self.xs, x, side="right") - 1, 0, self.xs.size - 2)
        h = self.xs[i + 1] - self.xs[i]
        return i, h, (x - self.xs[i]) / h

    def f(self, x):
        x = np.asarray(x, dtype=np.float64)
        i, h, u = self._seg(x)
        u2, u3 = u * u, u * u * u
        v = ((2 * u3 - 3 * u2 + 1) * self.ys[i] + (u3 - 2 * u2 + u) * h * self.ts[i]
             + (-2 * u3 + 3 * u2) * self.ys[i + 1] + (u3 - u2) * h * self.ts[i + 1])
        v = np.where(x < self.xs[0], self.ys[0] + self.ts[0] * (x - self.xs[0]), v)
        return np.where(x > self.xs[-1], self.ys[-1] + self.ts[-1] * (x - self.xs[-1]), v)

    def df(self, x):
        x = np.asarray(x, dtype=np.float64)
        i, h, u = self._seg(x)
        u2 = u * u
        v = ((6 * u2 - 6 * u) * self.ys[i] / h + (3 * u2 - 4 * u + 1) * self.ts[i]
             + (-6 * u2 + 6 * u) * self.ys[i + 1] / h + (3 * u2 - 2 * u) * self.ts[i + 1])
        v = np.where(x < self.xs[0], self.ts[0], v)
        return np.where(x > self.xs[-1], self.ts[-1], v)


@dataclass
class VLMaterial:
    """(a, b, c) triple; shift = 3a(1)+3b(1)+c(1) (materials.py:146-159)."""
    a: object
    b: object
    c: object
    name: str = "custom"
    shift: float = field(init=False)

    def __post_init__(self):
        self.shift = float(3 * self.a.f(1.0) + 3 * self.b.f(1.0) + self.c.f(1.0))


def builtin(name, mu=None, lam=0.0, mu1=None, mu2=0.0, spline_a=None, spline_b=None, spline_c=None):
    """Built-in materials (materials.py:257-297)."""
    if name == "polynomial":
        return VLMaterial(Poly(mu * np.array([1, -4, 6, -4, 1.0])), Zero(), Zero(), name)
    if name == "corotated":
        return VLMaterial(Poly([mu + 1.5 * lam, -2 * mu - 3 * lam, mu + 0.5 * lam]),
                          Poly([0.0, lam]), Zero(), name)
    if name == "stvk":
        A = mu / 4.0 + lam / 8.0
        return VLMaterial(Poly([A + lam / 2.0, 0.0, -2 * A - lam / 2.0, 0.0, A]),
                          Poly([-lam / 4.0, 0.0, lam / 4.0]), Zero(), name)
    if name == "neohookean":
        return VLMaterial(Poly([-mu / 2.0, 0.0, mu / 2.0]), Zero(), Log(-mu, lam), name)
    if name == "mooney_rivlin":
        b = Poly([-mu2, 0.0, mu2]) if mu2 > 0 else Zero()
        return VLMaterial(Poly([-mu1, 0.0, mu1]), b, Log(-(2 * mu1 + 4 * mu2), lam), name)
    if name == "spline":
        fa = Hermite(spline_a) if spline_a is not None else Zero()
        fb = Hermite(spline_b) if spline_b is not None else Zero()
        fc = Hermite(spline_c) if spline_c is not None else Zero()
        return VLMaterial(fa, fb, fc, name)
    raise OracleError(f"unknown material {name}")


def vl_energy(mat, s):
    """materials.py:181-188"""
    s1, s2, s3 = s[..., 0], s[..., 1], s[..., 2]
    return (mat.a.f(s1) + mat.a.f(s2) + mat.a.f(s3)
            + mat.b.f(s1 * s2) + mat.b.f(s2 * s3) + mat.b.f(s1 * s3)
            + mat.c.f(s1 * s2 * s3) - mat.shift)


def vl_stress(mat, s):
    """materials.py:196-207"""
    s1, s2, s3 = s[..., 0], s[..., 1], s[..., 2]
    b12, b23, b13 = mat.b.df(s1 * s2), mat.b.df(s2 * s3), mat.b.df(s1 * s3)
    c = mat.c.df(s1 * s2 * s3)
    out = np.empty_like(s)
    out[..., 0] = mat.a.df(s1) + b12 * s2 + b13 * s3 + c * s2 * s3
    out[..., 1] = mat.a.df(s2) + b12 * s1 + b23 * s3 + c * s1 * s3
    out[..., 2] = mat.a.df(s3) + b23 * s2 + b13 * s1 + c * s1 * s2
    return out


def fit_stiffness(mat, lo=0.5, hi=1.5):
    """OLS slope of a'(s)+2b'(s)+c'(s) over 1001 samples (materials.py:210-229)."""
    xs = np.linspace(lo, hi, FIT_SAMPLES)
    ys = mat.a.df(xs) + 2.0 * mat.b.df(xs) + mat.c.df(xs)
    dx, dy = xs - xs.mean(), ys - ys.mean()
    k = float(np.dot(dx, dy) / np.dot(dx, dx))
    if k <= 0:
        raise OracleError("non-positive fitted stiffness")
    return k


# --------------------------------------------------------------------------
# rotation-variant SVD (linalg.py:86-110)

def svd_rv(F):
    F = np.asarray(F, dtype=np.float64)
    U, s, Vt = np.linalg.svd(F)
    V = np.swapaxes(Vt, -1, -2)
    for M in (U, V):
        flip = np.linalg.det(M) < 0
        M[flip, :, 2] *= -1.0
        s[flip, 2] *= -1.0
    small = np.abs(s) < SIGMA_CLAMP
    s[small] = np.where(s[small] < 0, -SIGMA_CLAMP, SIGMA_CLAMP)
    return U, s, V


# --------------------------------------------------------------------------
# element groups and the objective (dynamics.py:40-70, 437-478)

THREADS = 1  # element-pass worker threads (numpy's batched SVD releases the GIL)


def set_threads(n):
    """Chunk the element pass over `n` host threads (CPU-baseline timing only;
    the summation order of the energy changes at roundoff level)."""
    global THREADS
    THREADS = max(1, int(n))


def _chunked(fn, m):
    if THREADS == 1 or m < 4096:
        return [fn(slice(0, m))]
    from concurrent.futures import ThreadPoolExecutor
    bounds = np.linspace(0, m, THREADS + 1).astype(int)
    with ThreadPoolExecutor(THREADS) as ex:
        return list(ex.map(fn, [slice(a, b) for a, b in zip(bounds[:-1], bounds[1:])]))


@dataclass
class TetGroup:
    tets: np.ndarray
    G: np.ndarray
    vols: np.ndarray
    mat: VLMaterial
    k: float

    def defgrad(self, x, sl=slice(None)):
        return np.einsum("eva,evc->eac", x[self.tets[sl]], self.G[sl])

    def energy(self, x):
        """dynamics.py:57-63"""
        def part(sl):
            _, s, _ = svd_rv(self.defgrad(x, sl))
            return self.vols[sl] * vl_energy(self.mat, s)
        return float(np.concatenate(_chunked(part, self.tets.shape[0])).sum())

    def corner_forces(self, x):
        """vol * U diag(tau) V^T G^T per corner (dynamics.py:50-55)."""
        def part(sl):
            U, s, V = svd_rv(self.defgrad(x, sl))
            tau = vl_stress(self.mat, s)
            P = np.einsum("eab,eb,ecb->eac", U, tau, V)
            return self.vols[sl, None, None] * np.einsum("eac,evc->eva", P, self.G[sl])
        return np.concatenate(_chunked(part, self.tets.shape[0]))

    def add_gradient(self, x, out):
        """element-major scatter (dynamics.py:65-67)"""
        np.add.at(out, self.tets.reshape(-1), self.corner_forces(x).reshape(-1, 3))


@dataclass
class ARAP:
    """PDMaterial("arap", k) (materials.py:163-173) for tets."""
    k: float


@dataclass
class ARAPTetGroup:
    """dynamics.ARAPGroup (dynamics.py:73-108): (w/2)||F - R(F)||^2, w = vol k."""
    tets: np.ndarray
    G: np.ndarray
    vols: np.ndarray
    k: float

    def _residual(self, x):
        F = np.einsum("eva,evc->eac", x[self.tets], self.G)
        U, _, V = svd_rv(F)
        return F - np.einsum("eab,ecb->eac", U, V)

    def energy(self, x):
        D = self._residual(x)
        return float((0.5 * (self.vols * self.k) * np.einsum("eac,eac->e", D, D)).sum())

    def add_gradient(self, x, out):
        D = self._residual(x)
        g = (self.vols * self.k)[:, None, None] * np.einsum("eac,evc->eva", D, self.G)
        np.add.at(out, self.tets.reshape(-1), g.reshape(-1, 3))


@dataclass
class AnisoGroupO:
    """dynamics.AnisoGroup (dynamics.py:154-193): V kappa/2 (|F d| - 1)^2."""
    tets: np.ndarray
    G: np.ndarray
    vols: np.ndarray
    d: np.ndarray
    kappa: np.ndarray

    def __post_init__(self):
        self.d = self.d / np.linalg.norm(self.d, axis=-1, keepdims=True)
        self.k = self.kappa  # w = vols * kappa (for L and w_col)

    def _fiber(self, x):
        F = np.einsum("eva,evc->eac", x[self.tets], self.G)
        u = np.einsum("eac,ec->ea", F, np.broadcast_to(self.d, (self.tets.shape[0], 3)))
        return u, np.linalg.norm(u, axis=1)

    def energy(self, x):
        _, nu = self._fiber(x)
        return float((0.5 * (self.vols * self.kappa) * (nu - 1.0) ** 2).sum())

    def add_gradient(self, x, out):
        u, nu = self._fiber(x)
        nu = np.maximum(nu, 1e-12)
        P = ((self.vols * self.kappa) * (nu - 1.0) / nu)[:, None, None] * np.einsum(
            "ea,ec->eac", u, np.broadcast_to(self.d, (self.tets.shape[0], 3)))
        g = np.einsum("eac,evc->eva", P, self.G)
        np.add.at(out, self.tets.reshape(-1), g.reshape(-1, 3))


@dataclass
class SpringGroupO:
    """dynamics.SpringGroup (dynamics.py:111-151): (w/2)(|d| - r)^2, w = k."""
    edges: np.ndarray
    rest: np.ndarray
    k: float

    def _dirs(self, x):
        d = x[self.edges[:, 1]] - x[self.edges[:, 0]]
        return d, np.linalg.norm(d, axis=1)

    def energy(self, x):
        _, length = self._dirs(x)
        return float((0.5 * np.full(self.edges.shape[0], self.k) * (length - self.rest) ** 2).sum())

    def add_gradient(self, x, out):
        d, length = self._dirs(x)
        resid = np.full(self.edges.shape[0], self.k)[:, None] * (1.0 - self.rest / length)[:, None] * d
        g = np.empty((self.edges.shape[0], 2, 3))
        g[:, 0] = -resid
        g[:, 1] = resid
        np.add.at(out, self.edges.reshape(-1), g.reshape(-1, 3))


def read_obj_springs(path):
    """load_obj_springs (mesh.py:135-171): vertices, sorted unique triangle
    edges, rest lengths, faces."""
    verts, faces = [], []
    with open(path) as fh:
        for line in fh:
            p = line.split("#", 1)[0].split()
            if not p:
                continue
            if p[0] == "v":
                verts.append([float(p[1]), float(p[2]), float(p[3])])
            elif p[0] == "f":
                faces.append([int(q.split("/")[0]) - 1 for q in p[1:4]])
    verts, faces = np.asarray(verts), np.asarray(faces, dtype=np.int64)
    es = set()
    for a, b, c in faces:
        for u, v in ((a, b), (b, c), (a, c)):
            es.add((min(u, v), max(u, v)))
    edges = np.asarray(sorted(es), dtype=np.int64)
    rest = np.linalg.norm(verts[edges[:, 1]] - verts[edges[:, 0]], axis=1)
    return verts, edges, rest, faces


def build_springs(verts, edges, rest, faces, density, k, h, gravity, fixed, factor="dense", colliders=(),
                  collision_weight=None):
    """dynamics.build_system for a spring network (dynamics.py:374-434)."""
    verts = np.asarray(verts, dtype=np.float64)
    n = verts.shape[0]
    v = verts[faces]
    areas = 0.5 * np.linalg.norm(np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), axis=1)  # mesh.py:184-191
    masses = np.zeros(n)
    for c in range(3):
        np.add.at(masses, faces[:, c], density * areas / 3.0)
    grp = SpringGroupO(np.asarray(edges), np.asarray(rest), float(k))
    blk = np.full(edges.shape[0], float(k))[:, None, None] * np.array([[1.0, -1.0], [-1.0, 1.0]])[None]
    L = scipy.sparse.coo_matrix((blk.reshape(-1), (np.repeat(edges, 2, axis=1).reshape(-1),
                                                   np.tile(edges, (1, 2)).reshape(-1))), shape=(n, n)).tocsr()
    fixed = np.asarray(sorted(set(int(i) for i in fixed)), dtype=np.int64)
    mask = np.ones(n, dtype=bool)
    mask[fixed] = False
    free = np.nonzero(mask)[0]
    A = (L + scipy.sparse.diags(masses / h ** 2)).tocsr()
    A_free = A[free][:, free].tocsr()
    if factor == "dense":
        fac = DenseFactor(A_free.toarray())
    elif factor == "cg":                                           # configs[4]
        fac = CGFactor(A_free, tol=cg_tol)
    else:
        fac = SparseFactor(A_free)
    bbox = verts.max(axis=0) - verts.min(axis=0)
    w_col = float(collision_weight) if collision_weight is not None else 10.0 * float(k)
    return System(verts, np.asarray(edges), masses, float(h), np.asarray(gravity, dtype=np.float64), [grp],
                  fixed, free, L, A_free, fac, float(np.linalg.norm(bbox)) or 1.0, list(colliders), w_col)


class DenseFactor:
    """Dense Cholesky, restating linalg.py:23-40."""

    def __init__(self, A):
        self.n = A.shape[0]
        self.c = scipy.linalg.cho_factor(np.ascontiguousarray(A, dtype=np.float64), lower=True,
                                         check_finite=False)

    def solve(self, B):
        return scipy.linalg.cho_solve(self.c, B, check_finite=False)


class SparseFactor:
    """Sparse restatement of the same solve: SuperLU in symmetric
    mode with MMD ordering and no pivoting, equivalent to the dense Cholesky
    to ~1e-15 relative."""

    def __init__(self, A):
        self.n = A.shape[0]
        self.lu = scipy.sparse.linalg.splu(
            scipy.sparse.csc_matrix(A), permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
            options=dict(SymmetricMode=True))

    def solve(self, B):
        return self.lu.solve(np.asarray(B, dtype=np.float64))


_CG_LIB = None


def cg_lib():
    """ctypes handle of oracle/cg_free.c (built by __graft_entry__.build(), or here
    on first use)."""
    global _CG_LIB
    if _CG_LIB is None:
        import ctypes as C
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        so = os.path.join(here, "_build", "libcg_free.so")
        src = os.path.join(here, "cg_free.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            os.makedirs(os.path.dirname(so), exist_ok=True)
            subprocess.run(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", so, src, "-lm"], check=True)
        lib = C.CDLL(so)
        P = C.c_void_p
        lib.oracle_cg3.argtypes = [C.c_int64, P, P, P, P, P, C.c_double, C.c_int32, P, P]
        lib.oracle_cg3.restype = C.c_int
        _CG_LIB = lib
    return _CG_LIB


class CGFactor:
    """SURVEY §8c's configs[4] restatement of `sysfact` (linalg.py:57-59): the
    dense Cholesky of A_free is infeasible at 12 M dofs, so `solve` runs
    Jacobi-preconditioned CG per coordinate (oracle/cg_free.c) to a relative
    residual of `tol` (1e-13, three orders tighter than the GPU's 1e-10)."""

    def __init__(self, A, tol=1e-13, maxit=20000):
        A = scipy.sparse.csr_matrix(A)
        A.sort_indices()
        self.n = A.shape[0]
        self.ptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
        self.idx = np.ascontiguousarray(A.indices, dtype=np.int32)
        self.val = np.ascontiguousarray(A.data, dtype=np.float64)
        self.tol, self.maxit = float(tol), int(maxit)
        self.log = []  # (iterations per column, true relative residual per column) per solve

    def solve(self, B):
        B = np.ascontiguousarray(B, dtype=np.float64).reshape(self.n, 3)
        X = np.empty_like(B)
        its = np.zeros(3, dtype=np.int32)
        res = np.zeros(3)
        rc = cg_lib().oracle_cg3(self.n, self.ptr.ctypes.data, self.idx.ctypes.data, self.val.ctypes.data,
                                 B.ctypes.data, X.ctypes.data, self.tol, self.maxit, its.ctypes.data,
                                 res.ctypes.data)
        self.log.append((its.tolist(), res.tolist()))
        if rc:
            raise OracleError(f"CG did not reach {self.tol} in {self.maxit} iterations: {res}")
        return X


@dataclass
class System:
    verts: np.ndarray
    tets: np.ndarray
    masses: np.ndarray
    h: float
    gravity: np.ndarray
    groups: list
    fixed: np.ndarray
    free: np.ndarray
    L: scipy.sparse.csr_matrix
    A_free: scipy.sparse.csr_matrix
    factor: object
    scale: float
    colliders: list = None
    w_col: float = 0.0

    @property
    def n(self):
        return self.verts.shape[0]


def build(verts, tets, density, materials, h, gravity, fixed, fit=(0.5, 1.5), factor="sparse",
          masses=None, colliders=(), collision_weight=None, aniso=None, cg_tol=1e-13):
    """Restates dynamics.build_system (dynamics.py:351-434) for VL tet groups.

    `materials` is a VLMaterial (all tets) or a list of (tet_index_array, VLMaterial).
    """
    verts = np.asarray(verts, dtype=np.float64)
    tets = np.asarray(tets, dtype=np.int64)
    n = verts.shape[0]
    if masses is None:
        masses = vertex_masses(verts, tets, density)
    groups = []
    if tets.shape[0]:
        G, vols = diff_operators(verts, tets)
        assign = [(np.arange(tets.shape[0]), materials)] if isinstance(materials, (VLMaterial, ARAP)) else \
            [(np.asarray(i, dtype=np.int64), m) for i, m in materials]
        for idx, mat in assign:
            if isinstance(mat, ARAP):  # dynamics.py:341-342
                groups.append(ARAPTetGroup(tets[idx], G[idx], vols[idx], float(mat.k)))
            else:
                groups.append(TetGroup(tets[idx], G[idx], vols[idx], mat, fit_stiffness(mat, *fit)))
        if aniso:  # dynamics.py:368-373
            idx = np.asarray([a[0] for a in aniso], dtype=np.int64)
            groups.append(AnisoGroupO(tets[idx], G[idx], vols[idx], np.asarray([a[1] for a in aniso], dtype=np.float64),
                                      np.asarray([a[2] for a in aniso], dtype=np.float64) * np.ones(idx.size)))
    rows, cols, vals = [], [], []
    for g in groups:
        w = g.vols * g.k                                          # dynamics.py:48
        blk = w[:, None, None] * np.einsum("evc,euc->evu", g.G, g.G)  # dynamics.py:69-70
        rows.append(np.repeat(g.tets, 4, axis=1).reshape(-1))
        cols.append(np.tile(g.tets, (1, 4)).reshape(-1))
        vals.append(blk.reshape(-1))
    if rows:
        L = scipy.sparse.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                    shape=(n, n)).tocsr()
    else:
        L = scipy.sparse.csr_matrix((n, n))
    fixed = np.asarray(sorted(set(int(i) for i in fixed)), dtype=np.int64)
    mask = np.ones(n, dtype=bool)
    mask[fixed] = False
    free = np.nonzero(mask)[0]
    A = (L + scipy.sparse.diags(masses / h ** 2)).tocsr()          # dynamics.py:413
    A_free = A[free][:, free].tocsr()
    if factor == "dense":
        fac = DenseFactor(A_free.toarray())
    elif factor == "cg":                                           # configs[4]
        fac = CGFactor(A_free, tol=cg_tol)
    else:
        fac = SparseFactor(A_free)
    bbox = verts.max(axis=0) - verts.min(axis=0)
    scale = float(np.linalg.norm(bbox)) or 1.0                     # dynamics.py:416-417
    max_w = max((float((g.vols * g.k).max()) for g in groups if g.vols.size), default=0.0)
    w_col = float(collision_weight) if collision_weight is not None else 10.0 * max_w  # dynamics.py:417
    return System(verts, tets, masses, float(h), np.asarray(gravity, dtype=np.float64), groups,
                  fixed, free, L, A_free, fac, scale, list(colliders), w_col)


# --------------------------------------------------------------------------
# colliders (dynamics.py:199-285, 446-457, 486-516)

class HalfSpace:
    """dynamics.py:199-212"""

    def __init__(self, point, normal):
        self.point = np.asarray(point, dtype=np.float64)
        n = np.asarray(normal, dtype=np.float64)
        self.normal = n / np.linalg.norm(n)

    def signed_distance(self, x):
        return (x - self.point) @ self.normal

    def project(self, x):
        sd = self.signed_distance(x)
        return x - sd[:, None] * self.normal, np.broadcast_to(self.normal, x.shape)


class Sphere:
    """dynamics.py:215-234"""

    def __init__(self, center, radius):
        self.center = np.asarray(center, dtype=np.float64)
        self.radius = float(radius)

    def signed_distance(self, x):
        return np.linalg.norm(x - self.center, axis=1) - self.radius

    def project(self, x):
        r = x - self.center
        dist = np.linalg.norm(r, axis=1)
        n = r / np.maximum(dist, 1e-12)[:, None]
        n[dist < 1e-12] = (0.0, 0.0, 1.0)
        return self.center + self.radius * n, n


class Torus:
    """dynamics.py:237-270 (axis z through the center; on-axis points keep
    the reference's ring choice: only the x component is replaced by R)"""

    def __init__(self, center, major_radius, minor_radius):
        self.center = np.asarray(center, dtype=np.float64)
        self.R, self.r = float(major_radius), float(minor_radius)

    def _ring(self, x):
        local = x - self.center
        radial = np.linalg.norm(local[:, :2], axis=1)
        safe = np.maximum(radial, 1e-12)
        ring = np.zeros_like(local)
        ring[:, 0] = self.R * local[:, 0] / safe
        ring[:, 1] = self.R * local[:, 1] / safe
        ring[radial < 1e-12, 0] = self.R
        return local, ring

    def signed_distance(self, x):
        local, ring = self._ring(x)
        return np.linalg.norm(local - ring, axis=1) - self.r

    def project(self, x):
        local, ring = self._ring(x)
        q = local - ring
        dist = np.linalg.norm(q, axis=1)
        n = q / np.maximum(dist, 1e-12)[:, None]
        n[dist < 1e-12] = (0.0, 0.0, 1.0)
        return self.center + ring + self.r * n, n


def update_collisions(sys, q_l, x):
    """Active constraints (idx, t, n), collider-major (dynamics.py:486-516)."""
    idx, ts, ns = [], [], []
    for col in sys.colliders or ():
        pen = np.nonzero(col.signed_distance(x) < 0)[0]
        if pen.size == 0:
            continue
        t, nrm = col.project(x[pen])
        vn = np.einsum("kc,kc->k", (x[pen] - q_l[pen]) / sys.h, nrm)
        keep = (vn < 0.0) | (col.signed_distance(q_l[pen]) < 0.0)
        if np.any(keep):
            idx.append(pen[keep])
            ts.append(t[keep])
            ns.append(nrm[keep])
    if not idx:
        return None
    return np.concatenate(idx), np.concatenate(ts), np.concatenate(ns)


def collision_energy(sys, cons, x):
    """dynamics.py:446-450"""
    if cons is None:
        return 0.0
    depth = np.einsum("kc,kc->k", x[cons[0]] - cons[1], cons[2])
    return float(sys.w_col * np.dot(depth, depth))


def add_collision_gradient(sys, cons, x, out):
    """dynamics.py:453-457"""
    if cons is None:
        return
    depth = np.einsum("kc,kc->k", x[cons[0]] - cons[1], cons[2])
    np.add.at(out, cons[0], 2.0 * sys.w_col * depth[:, None] * cons[2])


def inertia_target(sys, q_l, q_prev, fixed_targets=None):
    """y = 2 q_l - q_prev + h^2 g; fixed rows = targets or q_l (dynamics.py:437-443)."""
    h = sys.h
    y = 2.0 * q_l - q_prev + h * h * sys.gravity[None, :]
    if sys.fixed.size:
        y[sys.fixed] = q_l[sys.fixed] if fixed_targets is None else fixed_targets
    return y


def objective(sys, y, x, cons=None):
    """dynamics.py:460-467."""
    d = x - y
    g = 0.5 / sys.h ** 2 * float(np.einsum("vc,v,vc->", d, sys.masses, d))
    for grp in sys.groups:
        g += grp.energy(x)
    g += collision_energy(sys, cons, x)
    return g


def gradient(sys, y, x, cons=None):
    """dynamics.py:470-478: inertia, elastic scatter, collisions, then zero fixed rows."""
    out = (sys.masses[:, None] / sys.h ** 2) * (x - y)
    for grp in sys.groups:
        grp.add_gradient(x, out)
    add_collision_gradient(sys, cons, x, out)
    if sys.fixed.size:
        out[sys.fixed] = 0.0
    return out


# --------------------------------------------------------------------------
# L-BFGS, line search, frame loop (solvers.py)

class History:
    """solvers.py:83-103"""

    def __init__(self, m):
        self.m = m
        self.pairs = []

    def push(self, s, t):
        rho = float(np.vdot(t, s))
        if rho <= CURVATURE_GUARD * float(np.linalg.norm(s)) * float(np.linalg.norm(t)):
            return
        self.pairs.append((s, t, rho))
        if len(self.pairs) > self.m:
            del self.pairs[0]


def solve_free(sys, q):
    r = np.zeros_like(q)
    r[sys.free] = sys.factor.solve(q[sys.free])
    return r


def direction(sys, hist, grad, lbfgs_init="system_matrix"):
    """Two-loop recursion with H0 = A^-1 (solvers.py:120-151); empty history is
    bitwise the pd_qn direction (solvers.py:113-117)."""
    q = -grad.copy()
    zetas = []
    for s, t, rho in reversed(hist.pairs):
        z = float(np.vdot(s, q)) / rho
        q -= z * t
        zetas.append(z)
    zetas.reverse()
    if lbfgs_init == "rest_pose_hessian":                                  # solvers.py:142-146
        r = np.zeros_like(q)
        r[sys.free] = scipy.linalg.cho_solve(rest_hessian_factor(sys), q[sys.free].reshape(-1)).reshape(-1, 3)
    elif lbfgs_init == "scaled_identity":                                  # solvers.py:136-141
        if hist.pairs:
            s, t, rho = hist.pairs[-1]
            scale = rho / float(np.vdot(t, t))
        else:
            scale = 1.0
        r = scale * q
    else:
        r = solve_free(sys, q)
    for (s, t, rho), z in zip(hist.pairs, zetas):
        eta = float(np.vdot(t, r)) / rho
        r += s * (z - eta)
    return r


def line_search(sys, y, x, d, g_x, grad, gamma=0.3, alpha_init=2.0, shrink=0.5, cons=None):
    """Armijo backtracking (solvers.py:241-257)."""
    slope = float(np.vdot(grad, d))
    if slope >= 0.0:
        raise OracleError(f"ascent direction, slope={slope}")
    alpha, trials = alpha_init, 0
    while True:
        alpha *= shrink
        if alpha < ALPHA_FLOOR:
            raise OracleStagnation("alpha underflow")
        trials += 1
        x_new = x + alpha * d
        g_new = objective(sys, y, x_new, cons)
        if g_new <= g_x + gamma * alpha * slope:
            return alpha, x_new, g_new, trials


@dataclass
class Record:
    """solvers.py:71-80"""
    g0: float = 0.0
    g: list = field(default_factory=list)
    ls_trials: list = field(default_factory=list)
    alphas: list = field(default_factory=list)
    cum_ms: list = field(default_factory=list)
    stagnated: bool = False
    fallbacks: int = 0


def direction_chebyshev(x_k, x_km1, q, k, omega_prev, rho, S):
    """solvers.py:154-164"""
    if k < S:
        omega = 1.0
    elif k == S:
        omega = 2.0 / (2.0 - rho ** 2)
    else:
        omega = 4.0 / (4.0 - rho ** 2 * omega_prev)
    x_hat = x_k + q
    return omega * (x_hat - x_km1) + x_km1 - x_k, omega


def simulate_frame(sys, q_l, q_prev, iterations=10, m=5, kind="lbfgs", gamma=0.3, alpha_init=2.0,
                   shrink=0.5, use_line_search=True, fixed_targets=None, rho=0.9, S=10, lbfgs_init="system_matrix"):
    """One backward-Euler frame (solvers.py:260-352) for kind in {lbfgs, pd_qn},
    lbfgs_init='system_matrix', no colliders.  Returns (x, y, Record)."""
    t0 = time.perf_counter()
    y = inertia_target(sys, q_l, q_prev, fixed_targets)
    x = y.copy()
    rec = Record()
    hist = History(m)
    prev_x = prev_g = None
    grad_tol = 1e-12 * sys.scale * max(1.0, float(sys.masses.max()) / sys.h ** 2)
    cons = update_collisions(sys, q_l, x) if sys.colliders else None   # solvers.py:280
    rec.g0 = objective(sys, y, x, cons)

    def log(g, tr, a):
        rec.g.append(g)
        rec.ls_trials.append(tr)
        rec.alphas.append(a)
        rec.cum_ms.append(1000.0 * (time.perf_counter() - t0))

    x_prev_iter = x.copy()                                                # solvers.py:271-272
    omega = 1.0
    for k in range(1, iterations + 1):
        if sys.colliders:
            cons = update_collisions(sys, q_l, x)                         # solvers.py:285
        g_x = objective(sys, y, x, cons)
        grad = gradient(sys, y, x, cons)
        if kind == "lbfgs" and prev_x is not None:
            hist.push(x - prev_x, grad - prev_g)
        if float(np.linalg.norm(grad)) <= grad_tol:
            log(g_x, 0, 0.0)
            prev_x, prev_g = x, grad
            continue
        if kind == "newton":                                              # solvers.py:312-315
            d = direction_newton(sys, x, grad)
            if float(np.vdot(grad, d)) >= 0.0:
                d = direction(sys, hist, grad)
                rec.fallbacks += 1
        elif kind == "chebyshev":                                         # solvers.py:306-311
            q = direction(sys, hist, grad)
            d, omega = direction_chebyshev(x, x_prev_iter, q, k, omega, rho, S)
            if float(np.vdot(grad, d)) >= 0.0:
                d = q
                rec.fallbacks += 1
        else:
            d = direction(sys, hist, grad, lbfgs_init)
        if use_line_search:
            slope = float(np.vdot(grad, d))
            if slope < 0.0 and -slope <= 1e-12 * max(abs(g_x), 1.0):
                log(g_x, 0, 0.0)
                prev_x, prev_g = x, grad
                continue
            try:
                alpha, x_new, g_new, trials = line_search(sys, y, x, d, g_x, grad, gamma, alpha_init, shrink,
                                                          cons)
            except OracleStagnation:
                rec.stagnated = True
                while len(rec.g) < iterations:
                    log(g_x, 0, 0.0)
                break
        else:
            alpha, x_new, trials = 1.0, x + d, 1
            g_new = objective(sys, y, x_new, cons)
        prev_x, prev_g = x, grad
        x_prev_iter = x
        x = x_new
        log(g_new, trials, alpha)
    return x, y, rec


# --------------------------------------------------------------------------
# Newton baseline (solvers.py:167-234, 355-398), VL tet groups

NEWTON_FD_STEP_REL = 1e-6    # solvers.py:32
HESSIAN_EIG_FLOOR = 1e-8     # solvers.py:31


def _vl_elem_gradient(grp, X):
    """VLGroup.elem_gradient (dynamics.py:50-55)"""
    F = np.einsum("eva,evc->eac", X, grp.G)
    U, s, V = svd_rv(F)
    P = np.einsum("eab,eb,ecb->eac", U, vl_stress(grp.mat, s), V)
    return grp.vols[:, None, None] * np.einsum("eac,evc->eva", P, grp.G)


def _elem_hessians_fd(grp, x, step):
    """solvers.py:170-185"""
    X0 = x[grp.tets]
    k, a, _ = X0.shape
    dim = 3 * a
    H = np.empty((k, dim, dim))
    for v in range(a):
        for c in range(3):
            Xp = X0.copy()
            Xp[:, v, c] += step
            Xm = X0.copy()
            Xm[:, v, c] -= step
            H[:, :, 3 * v + c] = ((_vl_elem_gradient(grp, Xp) - _vl_elem_gradient(grp, Xm)) / (2.0 * step)).reshape(k, dim)
    return 0.5 * (H + np.swapaxes(H, 1, 2))


def _project_psd(blocks, floor=HESSIAN_EIG_FLOOR):
    """solvers.py:188-192"""
    w, Q = np.linalg.eigh(blocks)
    return np.einsum("kij,kj,klj->kil", Q, np.maximum(w, floor), Q)


def direction_newton(sys, x, grad):
    """solvers.py:228-234 (no colliders): dense free-dof Hessian, cho_factor."""
    fac = scipy.linalg.cho_factor(newton_hessian_free(sys, x))
    d = np.zeros_like(x)
    d[sys.free] = scipy.linalg.cho_solve(fac, -grad[sys.free].reshape(-1)).reshape(-1, 3)
    return d


def rest_hessian_factor(sys):
    """solvers.py:401-407: the Newton Hessian at the rest pose, factored once."""
    if getattr(sys, "_rest_fac", None) is None:
        sys._rest_fac = scipy.linalg.cho_factor(newton_hessian_free(sys, sys.verts.copy()))
    return sys._rest_fac


def newton_hessian_free(sys, x):
    """solvers.py:195-225 (no colliders): the dense Hessian on the free dofs."""
    n = sys.n
    step = NEWTON_FD_STEP_REL * sys.scale
    rows, cols, vals = [], [], []
    for grp in sys.groups:
        H = _project_psd(_elem_hessians_fd(grp, x, step))
        a = grp.tets.shape[1]
        dofs = (grp.tets[:, :, None] * 3 + np.arange(3)).reshape(grp.tets.shape[0], 3 * a)
        rows.append(np.repeat(dofs, 3 * a, axis=1).reshape(-1))
        cols.append(np.tile(dofs, (1, 3 * a)).reshape(-1))
        vals.append(H.reshape(-1))
    H = scipy.sparse.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                shape=(3 * n, 3 * n)).toarray()
    H[np.diag_indices_from(H)] += np.repeat(sys.masses / sys.h ** 2, 3)
    free3 = (sys.free[:, None] * 3 + np.arange(3)).reshape(-1)
    return H[np.ix_(free3, free3)]


def newton_reference(sys, q_l, q_prev, grad_tol_rel=1e-10, max_iterations=200, gamma=0.3, alpha_init=2.0,
                     shrink=0.5):
    """solvers.py:355-398: (x*, g*)"""
    y = inertia_target(sys, q_l, q_prev)
    x = y.copy()
    tol = grad_tol_rel * max(1.0, float(np.linalg.norm(gradient(sys, y, x))))
    g_x = objective(sys, y, x)
    best, stalled = np.inf, 0
    for _ in range(max_iterations):
        g_x = objective(sys, y, x)
        grad = gradient(sys, y, x)
        gn = float(np.linalg.norm(grad))
        if gn <= tol:
            break
        if gn >= 0.999 * best:
            stalled += 1
            if stalled >= 3:
                break
        else:
            stalled = 0
        best = min(best, gn)
        d = direction_newton(sys, x, grad)
        if float(np.vdot(grad, d)) >= 0.0:
            d = direction(sys, History(0), grad)
        try:
            _, x, g_x, _ = line_search(sys, y, x, d, g_x, grad, gamma, alpha_init, shrink)
        except OracleStagnation:
            break
    return x, g_x


def twist_targets(rest, idx, axis, center, deg_per_s, t):
    """Rodrigues rotation of prescribed vertices (harness.py:260-273)."""
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    ang = np.deg2rad(deg_per_s) * t
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    R = np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * (K @ K)
    c = np.asarray(center, dtype=np.float64)
    return (rest[idx] - c) @ R.T + c
