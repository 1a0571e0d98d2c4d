"""Backward-Euler system on the B200 (mirror of qnsim.dynamics, dynamics.py:1-516).

`build_system` keeps the reference signature and setup semantics
(dynamics.py:351-434): lumped masses, G operators, per-group stiffness fit
w = V k, L = sum w G G^T, fixed/free split, A = L + M/h^2 on the free DOFs
factored once.  The result is a device-resident `SimSystem` backed by the
C-ABI `qn_system` (tets SoA, vertex->element gather map, supernodal factor,
solver workspace, CUDA graph of the frame).  `build_batch_system` adds the
configs[3] case: many instances of one mesh with per-instance materials and
numeric factors.

Beyond the VL tet groups: ARAP tets run as a VL
material, spring networks (cloth) run the spring branch of the element kernel,
colliders (HalfSpace, SphereCollider, TorusCollider) run inside the frame
graph, anisotropic fibres run the fibre branch of the per-tet kernel.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse

from paper_1604_07378_b200 import _lib
from paper_1604_07378_b200.linalg import Factorization
from paper_1604_07378_b200.materials import AnisoMaterial, FitInterval, MaterialModel, PDMaterial, estimate_stiffness
from paper_1604_07378_b200.mesh import VOLUME_EPS, MeshError, SpringNetwork, TetMesh, lumped_masses, tet_diff_operators

DEFAULT_TIMESTEP = 1.0 / 30.0      # dynamics.py:28
DEFAULT_GRAVITY = (0.0, 0.0, -9.8)  # dynamics.py:29


class DynamicsError(Exception):
    pass


class VLGroup:
    """Valanis-Landel tet group; GPU seam with the reference duck type
    (`energy`, `add_gradient`, `L_blocks`, `w`, `verts`; dynamics.py:40-70)."""

    def __init__(self, tets, G, vols, material: MaterialModel, k: float):
        self.verts = tets
        self.G = G
        self.vols = vols
        self.material = material
        self.w = vols * k
        self._system = None
        self._index = 0
        self._inst = 0

    def L_blocks(self):
        return self.w[:, None, None] * np.einsum("evc,euc->evu", self.G, self.G), self.verts

    def energy(self, x) -> float:
        e = C.c_double(0.0)
        xs = _lib.f64(x)
        _lib.check(_lib.load().qn_system_elements(self._system._h, self._inst, self._index, _lib.ptr(xs),
                                                  C.byref(e), None, _lib.QN_MEM_HOST, None), "group energy")
        return e.value

    def add_gradient(self, x, out):
        e = C.c_double(0.0)
        xs = _lib.f64(x)
        buf = _lib.f64(out)
        _lib.check(_lib.load().qn_system_elements(self._system._h, self._inst, self._index, _lib.ptr(xs),
                                                  C.byref(e), _lib.ptr(buf), _lib.QN_MEM_HOST, None), "group grad")
        out[...] = buf


class SpringGroup(VLGroup):
    """Edge springs with the PD energy (w/2)(|d| - r)^2, w = k (dynamics.py:111-151);
    GPU seam with the same duck type."""

    def __init__(self, edges, rest, k: float):
        self.verts = edges
        self.rest = rest
        self.w = np.full(edges.shape[0], float(k))
        self._system, self._index, self._inst = None, 0, 0

    def L_blocks(self):
        block = np.array([[1.0, -1.0], [-1.0, 1.0]])
        return self.w[:, None, None] * block[None], self.verts


class HalfSpace:
    """dynamics.py:199-212: keeps vertices on the positive side of a plane."""

    def __init__(self, point, normal):
        self.point = np.asarray(point, dtype=np.float64)
        n = np.asarray(normal, dtype=np.float64)
        self.normal = n / np.linalg.norm(n)

    def signed_distance(self, x):
        return (x - self.point) @ self.normal

    def to_c(self):
        c = _lib.Collider()
        c.kind = _lib.QN_COL_HALFSPACE
        c.p[:], c.n[:] = self.point, self.normal
        return c


class SphereCollider:
    """dynamics.py:215-234: keeps vertices outside a solid sphere."""

    def __init__(self, center, radius):
        self.center = np.asarray(center, dtype=np.float64)
        self.radius = float(radius)

    def signed_distance(self, x):
        return np.linalg.norm(x - self.center, axis=1) - self.radius

    def to_c(self):
        c = _lib.Collider()
        c.kind = _lib.QN_COL_SPHERE
        c.p[:] = self.center
        c.r0 = self.radius
        return c


class TorusCollider:
    """dynamics.py:237-270: keeps vertices outside a solid torus (axis z)."""

    def __init__(self, center, major_radius, minor_radius):
        self.center = np.asarray(center, dtype=np.float64)
        self.R = float(major_radius)
        self.r = float(minor_radius)

    def to_c(self):
        c = _lib.Collider()
        c.kind = _lib.QN_COL_TORUS
        c.p[:] = self.center
        c.r0, c.r1 = self.R, self.r
        return c


@dataclass
class SimState:
    """dynamics.py:314-329.  `collisions` is the active contact set of the
    reference's host loop (CollisionSet: idx / t / n); the frame graph rebuilds
    its own set on the device (k_col), so only the objective / gradient seams
    look at this field (they refuse a non-empty set, see _objective_gradient)."""

    q_l: np.ndarray
    q_prev: np.ndarray
    y: np.ndarray | None = None
    collisions: object = None

    def copy(self):
        return SimState(self.q_l.copy(), self.q_prev.copy(), None if self.y is None else self.y.copy())


@dataclass
class SimSystem:
    mesh: object
    masses: np.ndarray
    h: float
    gravity: np.ndarray
    groups: list
    fixed: np.ndarray
    free: np.ndarray
    L: object
    sysfact: Factorization
    scale: float = 1.0
    n_inst: int = 1
    materials: list = field(default_factory=list)
    pd_groups: list = field(default_factory=list)
    colliders: list = field(default_factory=list)
    w_col: float = 0.0
    a_nnz: int = 0  # nonzeros of A_free (setup diagnostics)
    _h: object = None

    @property
    def n(self):
        return self.masses.shape[0]

    @property
    def n_free(self):
        return self.free.shape[0]

    @property
    def op_handle(self) -> int:
        """Integer handle for the torch custom ops (torch_ops.py)."""
        return int(self._h.value)

    def set_precision(self, precision: str):
        """"fp64" (default) or "fp32": the optional single-precision element
        pass (configs[2]); everything else stays fp64."""
        if precision not in ("fp64", "fp32"):
            raise DynamicsError(f"precision {precision!r}: fp64 | fp32")
        _lib.check(_lib.load().qn_system_set_precision(self._h, 1 if precision == "fp32" else 0), "set_precision")
        self.precision = precision

    def set_fault(self, mode: int, iteration: int = 1):
        """Test-only fault injection into the device line search (qn_system_set_fault):
        0 off, 1 ascent direction, 2 steps that only increase g (stagnation)."""
        _lib.check(_lib.load().qn_system_set_fault(self._h, int(mode), int(iteration)))

    def set_graph_mode(self, on: bool):
        _lib.check(_lib.load().qn_system_set_graph_mode(self._h, 1 if on else 0))

    def factor_info(self) -> dict:
        if self.sysfact is not None:
            return self.sysfact.info()
        amg = self.amg_info()
        return {"solver": "amg", **amg} if amg["levels"] else {"solver": "pcg"}

    def amg_info(self) -> dict:
        """AMG systems: number of levels, rows per level, host setup time."""
        out = np.zeros(42, dtype=np.int64)
        _lib.check(_lib.load().qn_system_amg_info(self._h, _lib.ptr(out), C.c_int64(out.size)))
        nl = int(out[0])
        nnz = out[12:12 + 3 * nl].reshape(nl, 3) if nl else np.zeros((0, 3), dtype=np.int64)
        return {"levels": nl, "rows": [int(v) for v in out[1:1 + nl]], "setup_s": out[11] / 1000.0,
                "nnz_A": [int(v) for v in nnz[:, 0]], "nnz_P": [int(v) for v in nnz[:, 1]],
                "nnz_R": [int(v) for v in nnz[:, 2]]}

    def time_kernel(self, kernel: str, reps: int = 20, stream=None) -> float:
        """Mean CUDA-event time (ms) of one stand-alone launch of a hot kernel:
        "tet" (per-tet pass at the resident q_l), "solve" (fwd+bwd SpTRSV) or
        "spmv" (the CG's A_free SpMV, PCG/AMG systems) or "vcycle" (one AMG
        V(1,1) preconditioner application on the resident level vectors)."""
        ms = C.c_double(0.0)
        _lib.check(_lib.load().qn_system_time_kernel(self._h, {"tet": 0, "solve": 1, "spmv": 2, "vcycle": 3}[kernel], reps,
                                                     C.byref(ms),
                                                     stream), "time_kernel")
        return ms.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.load().qn_system_destroy(h)
            except Exception:
                pass
            self._h = None


def _assign(mesh, materials):
    """Tet groups of a material assignment (dynamics.py:330-345); ARAP PD
    materials become their Valanis-Landel form (materials.PDMaterial.as_vl)."""
    if isinstance(materials, PDMaterial):
        materials = materials.as_vl()
    if isinstance(materials, MaterialModel):
        return [(np.arange(mesh.tets.shape[0]), materials)]
    out = []
    for idx, mat in materials:
        if isinstance(mat, PDMaterial):
            mat = mat.as_vl()
        if not isinstance(mat, MaterialModel):
            raise NotImplementedError(f"material {mat!r}: only Valanis-Landel tet groups run on the B200 path")
        out.append((np.asarray(idx, dtype=np.int64), mat))
    return out


def _aniso_groups(mesh, aniso):
    """(element_index, direction, kappa) triples -> one fibre group per distinct
    (direction, kappa), in order of first appearance, elements in list order."""
    keyed = {}
    for e, d, kappa in aniso:
        e = int(e)
        if not 0 <= e < mesh.tets.shape[0]:
            raise DynamicsError(f"anisotropy element {e} out of range")
        dn = np.asarray(d, dtype=np.float64)
        dn = dn / np.linalg.norm(dn)
        if float(kappa) < 0:
            raise DynamicsError("anisotropic stiffness must be non-negative")
        key = (float(dn[0]), float(dn[1]), float(dn[2]), float(kappa))
        keyed.setdefault(key, []).append(e)
    return [(np.asarray(idx, dtype=np.int64), AnisoMaterial(key[:3], key[3])) for key, idx in keyed.items()]


def _build(mesh, inst_materials, h, gravity, fixed, fit_interval, n_mat_groups, solver="direct", pcg_tol=1e-10,
           pcg_maxit=20000, colliders=(), collision_weight=None):
    if not isinstance(mesh, TetMesh):
        raise NotImplementedError("spring networks (cloth) are outside the B200 hot path")
    _lib.require_gpu()
    from paper_1604_07378_b200 import setup as dsetup
    import time as _time
    _t0 = _time.perf_counter()
    _tm = {}
    n = mesh.n
    device = dsetup.use_device(mesh.tets.shape[0], len(inst_materials))
    if not device:
        masses = lumped_masses(mesh)
        G, vols = tet_diff_operators(mesh)
    fixed = np.asarray(sorted(set(int(i) for i in fixed)), dtype=np.int64)
    if fixed.size and (fixed.min() < 0 or fixed.max() >= n):
        raise DynamicsError("fixed vertex index out of range")
    mask = np.ones(n, dtype=bool)
    mask[fixed] = False
    free = np.nonzero(mask)[0]
    if free.size == 0:
        raise DynamicsError("all vertices fixed; nothing to simulate")

    # group-major tet order = the reference's scatter order over groups
    assign0 = inst_materials[0]
    order = np.concatenate([idx for idx, _ in assign0]) if assign0 else np.zeros(0, dtype=np.int64)
    tet_mat = np.concatenate([np.full(idx.size, g, dtype=np.int32) for g, (idx, _) in enumerate(assign0)]) \
        if assign0 else np.zeros(0, dtype=np.int32)
    identity = order.size == mesh.tets.shape[0] and np.array_equal(order, np.arange(order.size))
    tets = mesh.tets if identity else mesh.tets[order]
    m = tets.shape[0]
    dev = None
    if device:  # configs[4]-size meshes: G, volumes, masses, L and A_free assembled on the GPU (setup.py)
        ks0 = [mat.k_fit if mat.k_fit is not None else estimate_stiffness(mat, fit_interval) for _, mat in assign0]
        Gs, vs, masses, L_dev, Af_dev = dsetup.assemble(mesh.vertices, tets, mesh.density,
                                                        np.asarray(ks0)[tet_mat], h, fixed, VOLUME_EPS)
        bad = np.nonzero(masses <= 0)[0]
        if bad.size:
            raise MeshError(f"vertex {bad[0]} has zero mass (isolated vertex?)")
        inv = np.empty_like(order)
        inv[order] = np.arange(order.size)
        G, vols = (Gs, vs) if identity else (Gs[inv], vs[inv])
        dev = (L_dev, Af_dev)
        _tm["device_assembly"] = _time.perf_counter() - _t0
    else:
        Gs, vs = (G, vols) if identity else (G[order], vols[order])

    # L = sum_groups w G G^T per instance, assembled exactly as the reference
    # does (COO in group-major order -> CSR, dynamics.py:387-402, so L is bitwise
    # the reference's), then A = L + M/h^2 restricted to the free dofs (:413-414)
    if not device:
        GG = np.einsum("evc,euc->evu", Gs, Gs) if m else np.zeros((0, 4, 4))
        rows = np.repeat(tets, 4, axis=1).reshape(-1)
        cols = np.tile(tets, (1, 4)).reshape(-1)
    diag_m = scipy.sparse.diags(masses / h ** 2)
    values, Ls, groups_per_inst, mats = [], [], [], []
    f_indptr = a_idx = None
    for assign in inst_materials:
        ks, gl = [], []
        for g, (idx, mat) in enumerate(assign):
            k = mat.k_fit if mat.k_fit is not None else estimate_stiffness(mat, fit_interval)
            ks.append(k)
            gl.append(VLGroup(mesh.tets[idx], G[idx], vols[idx], mat, k))
        if dev is not None:
            L, Af = dev
        else:
            w = (vs * np.asarray(ks)[tet_mat]) if m else np.zeros(0)
            L = scipy.sparse.coo_matrix(((w[:, None, None] * GG).reshape(-1), (rows, cols)), shape=(n, n)).tocsr() \
                if m else scipy.sparse.csr_matrix((n, n))
            Af = (L + diag_m).tocsr()[free][:, free].tocsr()
            Af.sort_indices()
        if f_indptr is None:
            f_indptr, a_idx = Af.indptr.astype(np.int64), Af.indices
        elif not (np.array_equal(f_indptr, Af.indptr) and np.array_equal(a_idx, Af.indices)):
            raise DynamicsError("instances must share the system-matrix pattern")
        Ls.append(L)
        values.append(Af.data)
        groups_per_inst.append(gl)
        mats.append([mat for _, mat in assign])
    fc = a_idx
    a_values = np.concatenate(values)
    a_indices = _lib.i32(fc)

    n_inst = len(inst_materials)
    n_mat = max(1, n_mat_groups)
    cmats = (_lib.Material * (n_inst * n_mat))()
    for b, ml in enumerate(mats):
        for g, mat in enumerate(ml):
            cmats[b * n_mat + g] = mat.to_c()

    tets32 = _lib.i32(tets)
    # Dm^-1 = G[:, 1:]: passed in place (stride 12) when G is contiguous, no copy
    if m and Gs.dtype == np.float64 and Gs.flags.c_contiguous:
        dminv, dminv_stride = Gs[:, 1:, :], 12
    else:
        dminv, dminv_stride = (_lib.f64(Gs[:, 1:, :]) if m else np.zeros((0, 3, 3))), 9
    vols_c = _lib.f64(vs)
    tm = _lib.i32(tet_mat) if n_mat > 1 else None
    masses_c = _lib.f64(masses)
    fixed32 = _lib.i32(fixed)
    f_indptr = _lib.i64(f_indptr)
    a_values = _lib.f64(a_values)
    coords = _lib.f64(mesh.vertices[free])
    bbox = mesh.vertices.max(axis=0) - mesh.vertices.min(axis=0)
    scale = float(np.linalg.norm(bbox)) or 1.0  # dynamics.py:416-417

    d = _lib.SystemDesc()
    d.n_verts, d.n_tets, d.n_inst, d.n_mat = n, m, n_inst, n_mat
    d.tets, d.vols = _lib.ptr(tets32), _lib.ptr(vols_c)
    d.Dm_inv = dminv.ctypes.data if m else None
    d.dminv_stride = dminv_stride
    d.tet_mat = _lib.ptr(tm)
    d.mats = C.cast(cmats, C.c_void_p)
    d.masses = _lib.ptr(masses_c)
    d.n_fixed, d.fixed = fixed.size, _lib.ptr(fixed32)
    d.h = float(h)
    for a in range(3):
        d.gravity[a] = float(gravity[a])
    d.scale = scale
    d.a_nnz = a_indices.size
    d.a_indptr, d.a_indices, d.a_values = _lib.ptr(f_indptr), _lib.ptr(a_indices), _lib.ptr(a_values)
    d.free_coords = _lib.ptr(coords)
    if solver not in ("direct", "pcg", "amg"):
        raise DynamicsError(f"unknown solver {solver!r} (direct | pcg | amg)")
    d.solver = {"direct": 0, "pcg": 1, "amg": 2}[solver]
    d.pcg_tol, d.pcg_maxit = float(pcg_tol), int(pcg_maxit)
    colliders = list(colliders)
    if len(colliders) > _lib.QN_MAX_COLLIDERS:
        raise DynamicsError(f"at most {_lib.QN_MAX_COLLIDERS} colliders")
    for col in colliders:
        if not hasattr(col, "to_c"):
            raise DynamicsError(f"unknown collider {col!r}")
    ccols = (_lib.Collider * max(1, len(colliders)))(*[col.to_c() for col in colliders])
    max_w = max((float(grp.w.max()) for gl in groups_per_inst for grp in gl if grp.w.size), default=0.0)
    w_col = float(collision_weight) if collision_weight is not None else 10.0 * max_w  # dynamics.py:417
    d.n_colliders, d.colliders, d.w_col = len(colliders), C.cast(ccols, C.c_void_p), w_col
    handle = C.c_void_p()
    _tm["host_prep"] = _time.perf_counter() - _t0 - sum(_tm.values())
    _lib.check(_lib.load().qn_system_create(C.byref(d), C.byref(handle)), "build_system")
    _tm["system_create"] = _time.perf_counter() - _t0 - sum(_tm.values())
    sysfact = None
    if solver == "direct":
        fh = C.c_void_p()
        _lib.check(_lib.load().qn_system_factor(handle, C.byref(fh)))
        sysfact = Factorization._borrow(fh, free.size, n_inst)

    system = SimSystem(mesh=mesh, masses=masses, h=float(h), gravity=np.asarray(gravity, dtype=np.float64),
                       groups=groups_per_inst[0] if n_inst == 1 else groups_per_inst, fixed=fixed, free=free,
                       L=Ls[0] if n_inst == 1 else Ls, sysfact=sysfact, scale=scale, n_inst=n_inst,
                       materials=mats, a_nnz=int(a_indices.size), colliders=colliders, w_col=w_col, _h=handle)
    for b, gl in enumerate(groups_per_inst):
        for g, grp in enumerate(gl):
            grp._system, grp._index, grp._inst = system, g, b
    system.build_times = _tm  # seconds per build phase (diagnostics)
    return system


def _build_springs(mesh: SpringNetwork, material, h, gravity, fixed, solver, pcg_tol, pcg_maxit, colliders,
                   collision_weight):
    """Spring-network system (dynamics.py:374-380 + the common assembly
    :382-434): one SpringGroup, L = sum w [[1,-1],[-1,1]], A = L + M/h^2 on the
    free vertices; the per-element pass runs the spring branch of the element
    kernel (elements (a, b, -1, -1), vols = rest lengths)."""
    if not isinstance(material, PDMaterial) or material.kind != "mass_spring":
        raise DynamicsError("spring networks require a mass_spring material")
    _lib.require_gpu()
    n, edges, rest = mesh.n, np.asarray(mesh.edges, dtype=np.int64), np.asarray(mesh.rest_lengths, np.float64)
    masses = lumped_masses(mesh)
    grp = SpringGroup(edges, rest, material.k)
    blocks, verts = grp.L_blocks()
    rows = np.repeat(verts, 2, axis=1).reshape(-1)
    cols = np.tile(verts, (1, 2)).reshape(-1)
    L = scipy.sparse.coo_matrix((blocks.reshape(-1), (rows, cols)), shape=(n, n)).tocsr()  # dynamics.py:398-402
    fixed = np.asarray(sorted(set(int(i) for i in fixed)), dtype=np.int64)
    if fixed.size and (fixed.min() < 0 or fixed.max() >= n):
        raise DynamicsError("fixed vertex index out of range")
    mask = np.ones(n, dtype=bool)
    mask[fixed] = False
    free = np.nonzero(mask)[0]
    if free.size == 0:
        raise DynamicsError("all vertices fixed; nothing to simulate")
    A = (L + scipy.sparse.diags(masses / h ** 2)).tocsr()
    Af = A[free][:, free].tocsr()
    Af.sort_indices()
    elems = np.full((edges.shape[0], 4), -1, dtype=np.int32)
    elems[:, :2] = edges
    cm = (_lib.Material * 1)()
    cm[0].a.kind, cm[0].a.c[0] = _lib.QN_FN_ZERO, float(material.k)
    bbox = mesh.vertices.max(axis=0) - mesh.vertices.min(axis=0)
    scale = float(np.linalg.norm(bbox)) or 1.0
    colliders = list(colliders)
    ccols = (_lib.Collider * max(1, len(colliders)))(*[col.to_c() for col in colliders])
    w_col = float(collision_weight) if collision_weight is not None else 10.0 * float(material.k)
    keep = (elems, _lib.f64(rest), _lib.f64(masses), _lib.i32(fixed), _lib.i64(Af.indptr), _lib.i32(Af.indices),
            _lib.f64(Af.data), _lib.f64(mesh.vertices[free]))
    d = _lib.SystemDesc()
    d.n_verts, d.n_tets, d.n_inst, d.n_mat = n, edges.shape[0], 1, 1
    d.tets, d.Dm_inv, d.vols, d.tet_mat = _lib.ptr(keep[0]), None, _lib.ptr(keep[1]), None
    d.mats = C.cast(cm, C.c_void_p)
    d.masses = _lib.ptr(keep[2])
    d.n_fixed, d.fixed = fixed.size, _lib.ptr(keep[3])
    d.h = float(h)
    for a in range(3):
        d.gravity[a] = float(gravity[a])
    d.scale = scale
    d.a_nnz = Af.nnz
    d.a_indptr, d.a_indices, d.a_values = _lib.ptr(keep[4]), _lib.ptr(keep[5]), _lib.ptr(keep[6])
    d.free_coords = _lib.ptr(keep[7])
    if solver not in ("direct", "pcg", "amg"):
        raise DynamicsError(f"unknown solver {solver!r} (direct | pcg | amg)")
    d.solver = {"direct": 0, "pcg": 1, "amg": 2}[solver]
    d.pcg_tol, d.pcg_maxit = float(pcg_tol), int(pcg_maxit)
    d.n_colliders, d.colliders, d.w_col = len(colliders), C.cast(ccols, C.c_void_p), w_col
    d.element_kind = _lib.QN_ELEM_SPRING
    handle = C.c_void_p()
    _lib.check(_lib.load().qn_system_create(C.byref(d), C.byref(handle)), "build_system")
    sysfact = None
    if solver == "direct":
        fh = C.c_void_p()
        _lib.check(_lib.load().qn_system_factor(handle, C.byref(fh)))
        sysfact = Factorization._borrow(fh, free.size, 1)
    system = SimSystem(mesh=mesh, masses=masses, h=float(h), gravity=np.asarray(gravity, dtype=np.float64),
                       groups=[grp], fixed=fixed, free=free, L=L, sysfact=sysfact, scale=scale, n_inst=1,
                       materials=[[material]], pd_groups=[grp], a_nnz=int(Af.nnz), colliders=colliders,
                       w_col=w_col, _h=handle)
    grp._system = system
    return system


def build_system(mesh, materials, h: float = DEFAULT_TIMESTEP, gravity=DEFAULT_GRAVITY, fixed=(), aniso=None,
                 colliders=(), collision_weight: float | None = None,
                 fit_interval: FitInterval = FitInterval(), solver: str = "direct", pcg_tol: float = 1e-10,
                 pcg_maxit: int = 20000, precision: str = "fp64") -> SimSystem:
    """dynamics.py:351-434 for Valanis-Landel tet groups (single instance).

    solver="direct" prefactors A_free once (the reference's semantics);
    solver="pcg" solves every direction with Jacobi-preconditioned CG to
    ||r|| <= pcg_tol ||b|| (configs[4]: meshes too large to factor);
    solver="amg" uses CG preconditioned by a smoothed-aggregation AMG V-cycle
    (same tolerance, ~40x fewer iterations on configs[4]).

    Inputs may be the reference's own objects (qnsim TetMesh / SpringNetwork,
    MaterialModel / PDMaterial, FitInterval, colliders): they are converted by
    `adopt` so that `qnsim.harness.build_system` can be swapped for this one."""
    from paper_1604_07378_b200 import adopt
    mesh, materials = adopt.mesh(mesh), adopt.materials(materials)
    fit_interval = adopt.fit_interval(fit_interval)
    colliders = [adopt.collider(c) for c in (colliders or ())]
    if isinstance(mesh, SpringNetwork):
        if aniso:
            raise DynamicsError("anisotropy applies to tet meshes only")
        return _build_springs(mesh, materials, h, gravity, fixed, solver, pcg_tol, pcg_maxit, colliders,
                              collision_weight)
    assign = _assign(mesh, materials)
    if aniso:  # AnisoGroup appended after the material groups (dynamics.py:368-373)
        assign = assign + _aniso_groups(mesh, aniso)
    system = _build(mesh, [assign], h, gravity, fixed, fit_interval, len(assign), solver, pcg_tol, pcg_maxit,
                    colliders, collision_weight)
    if precision != "fp64":
        system.set_precision(precision)
    return system


def build_batch_system(mesh, materials_per_instance, h: float = DEFAULT_TIMESTEP, gravity=DEFAULT_GRAVITY, fixed=(),
                       fit_interval: FitInterval = FitInterval(), colliders=(),
                       collision_weight: float | None = None) -> SimSystem:
    """configs[3]: independent instances of one mesh, one MaterialModel (or
    group assignment) per instance, each with its own factored A."""
    from paper_1604_07378_b200 import adopt
    mesh, fit_interval = adopt.mesh(mesh), adopt.fit_interval(fit_interval)
    colliders = [adopt.collider(c) for c in (colliders or ())]
    inst = [_assign(mesh, adopt.materials(m)) for m in materials_per_instance]
    if not inst:
        raise DynamicsError("empty batch")
    sizes = {len(a) for a in inst}
    if len(sizes) != 1:
        raise DynamicsError("all instances need the same material-group layout")
    return _build(mesh, inst, h, gravity, fixed, fit_interval, len(inst[0]), colliders=colliders,
                  collision_weight=collision_weight)


def inertia_target(state: SimState, system: SimSystem, fixed_targets=None) -> np.ndarray:
    """y = 2 q_l - q_prev + h^2 g (dynamics.py:437-443).  Host helper for API
    parity; the frame computes y on the device (k_init)."""
    h = system.h
    y = 2.0 * state.q_l - state.q_prev + h * h * system.gravity
    if system.fixed.size:
        if fixed_targets is None:
            y[..., system.fixed, :] = state.q_l[..., system.fixed, :]
        else:
            y[..., system.fixed, :] = fixed_targets
    return y


def _objective_gradient(system: SimSystem, state: SimState, x, want_grad: bool):
    cons = getattr(state, "collisions", None)
    if cons is not None and int(getattr(cons, "count", len(getattr(cons, "idx", ())))) > 0:
        # dynamics.py:464-467,475 add w_col * depth^2 terms for the active set; the
        # device seam evaluates inertia + elastic only, so a non-empty set would
        # silently differ from the reference
        raise NotImplementedError("objective/gradient seam: non-empty state.collisions (the contact penalty is "
                                  "evaluated inside simulate_frame's graph, not by this seam)")
    x = _lib.f64(x)
    y = _lib.f64(state.y)
    g = np.empty(system.n_inst)
    grad = np.empty_like(x) if want_grad else None
    _lib.check(_lib.load().qn_system_objective(system._h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(g), _lib.ptr(grad),
                                               _lib.QN_MEM_HOST, None), "objective")
    return g, grad


def objective(system: SimSystem, state: SimState, x) -> float:
    """g(x) = inertia + elastic on the GPU (dynamics.py:460-467)."""
    g, _ = _objective_gradient(system, state, x, False)
    return float(g[0]) if system.n_inst == 1 else g


def gradient(system: SimSystem, state: SimState, x) -> np.ndarray:
    """Gradient with fixed rows zeroed, on the GPU (dynamics.py:470-478)."""
    return _objective_gradient(system, state, x, True)[1]
