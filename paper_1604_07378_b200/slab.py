"""Slab-decomposed frame for one large mesh across ranks (configs[4]).

The reference has one process and one `simulate_frame` (solvers.py:260-352).
Here the mesh is cut into slabs of grid cells along x (`slab_layout`: the
cells balanced like `parallel.shard_instances`), one per rank; every rank keeps a one-cell ghost layer so that the
gradient of each owned vertex is computed locally, bit for bit as in the
single system, and the frame control (push, two-loop, CG, Armijo) runs on
global sums.  The device work is the C-ABI `qn_slab_*` stages
(paper_1604_07378_b200/csrc/qn_slab.cu); this module only
* builds each rank's slab-local system (`SlabRank`),
* moves data between ranks (`NcclComm`: NCCL all-gather of the stages'
  partial sums and send/recv of the boundary planes; `EmulatedComm`: the same
  exchanges between several slabs held by one process on one device, used to
  test the decomposition without more GPUs — no kernel ever waits on another
  rank's kernel, everything is stream-ordered), and
* runs the reference's frame control on the gathered scalars (`SlabRun`).

Scalars: each stage leaves this rank's fixed-order partial sums in SEND; the
all-gather puts every rank's SEND into GATHER ([ranks][32]); device kernels and
the host add the ranks in index order, so every rank takes the same decisions
and the emulated and multi-GPU runs produce the same numbers.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse

from paper_1604_07378_b200 import _lib
from paper_1604_07378_b200.dynamics import _build, DynamicsError
from paper_1604_07378_b200.materials import FitInterval, MaterialModel
from paper_1604_07378_b200.mesh import TetMesh, grid_bar_cells, lumped_masses
from paper_1604_07378_b200.parallel import shard_instances
from paper_1604_07378_b200.solvers import ConvergenceRecord, SolverConfig, SolverError

SEND, GATHER, P, R0, QL, QPREV, Y, X, G, CSEND, CGATHER = range(11)
(INIT, EVAL, GRAD, PCG_SETUP, PCG_P, PCG_SPMV, PCG_UPDATE, STORE, ETA, DIR, TRIAL, FINISH, PCG_RZ, COARSE_R,
 COARSE_APPLY) = range(15)
MAX_M = 8                 # kSlabMaxM
RING = MAX_M + 1
NSEND = 32
_STAGE_NAMES = ["init", "eval", "grad", "pcg_setup", "pcg_p", "pcg_spmv", "pcg_update", "store", "eta", "dir",
                "trial", "finish", "pcg_rz", "coarse_r", "coarse_apply"]
CURVATURE_GUARD = 1e-12   # solvers.py:28
ALPHA_FLOOR = 1e-12       # solvers.py:29


@dataclass
class SlabLayout:
    """Rank `rank`'s part of an (nx, ny, nz) Freudenthal bar (vertex id
    (i (ny+1) + j)(nz+1) + k, 6 tets per cell, cells x-major)."""
    grid: tuple
    world: int
    rank: int
    c0: int          # own cells [c0, c1)
    c1: int
    cl: int          # first local cell (c0 - 1 with a ghost layer)
    plane: int       # vertices per grid plane
    n: int           # local vertices: planes [cl, c1]
    own_lo: int      # owned local vertex range
    own_hi: int
    tet_own_lo: int  # local tets [tet_own_lo, m) are owned

    @property
    def v0(self):
        """global id of local vertex 0"""
        return self.cl * self.plane

    @property
    def tets_per_cell(self):
        return 6 * self.grid[1] * self.grid[2]


def slab_layout(grid, world: int, rank: int) -> SlabLayout:
    nx, ny, nz = grid
    if world > nx:
        raise ValueError(f"{world} slabs need at least {world} cells along x (have {nx})")
    c0, c1 = shard_instances(nx, world, rank)
    cl = c0 - 1 if rank > 0 else c0
    plane = (ny + 1) * (nz + 1)
    n = (c1 - cl + 1) * plane
    own_lo = (c0 - cl) * plane
    own_hi = n if rank == world - 1 else (c1 - cl) * plane
    return SlabLayout(tuple(grid), world, rank, c0, c1, cl, plane, n, own_lo, own_hi,
                      (c0 - cl) * 6 * ny * nz)


def local_tets_from_global(tets, lay: SlabLayout):
    per = lay.tets_per_cell
    return tets[lay.cl * per: lay.c1 * per] - lay.v0


def local_tets_generated(lay: SlabLayout, size):
    """The slab's tets without materialising the global mesh (configs[4])."""
    nx, ny, nz = lay.grid
    return grid_bar_cells(nx, ny, nz, size, lay.cl, lay.c1) - lay.v0


def slab_operator(L, masses, h, pin, owned):
    """A = L + M/h^2 (dynamics.py:398-414) on the owned free rows of a slab, in
    increasing local order, with the local non-pinned vertices as columns
    (column index = local vertex id): every owned row is complete because all
    its incident tets are local, so these rows are rows of the global A_free."""
    A = (L + scipy.sparse.diags(masses / h ** 2)).tocsr()
    A.sort_indices()
    rows = np.nonzero(owned & ~pin)[0]
    Ar = A[rows].tocoo()
    keep = ~pin[Ar.col]
    Ar = scipy.sparse.csr_matrix((Ar.data[keep], (Ar.row[keep], Ar.col[keep])), shape=(rows.size, A.shape[1]))
    Ar.sort_indices()
    return Ar


def stiffness_matrix(mesh, w):
    """L = sum_e w_e G_e G_e^T (dynamics.py:387-402) as CSR (host, setup)."""
    from paper_1604_07378_b200.mesh import tet_diff_operators
    G_, _ = tet_diff_operators(mesh)
    GG = np.einsum("evc,euc->evu", G_, G_) * np.asarray(w)[:, None, None]
    rows = np.repeat(mesh.tets, 4, axis=1).reshape(-1)
    cols = np.tile(mesh.tets, (1, 4)).reshape(-1)
    return scipy.sparse.csr_matrix((GG.reshape(-1), (rows, cols)), shape=(mesh.n, mesh.n))


class _CudaBuffer:
    """__cuda_array_interface__ view of a device buffer owned by the library."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class SlabRank:
    """One rank's slab: the slab-local system (own + ghost cells; ghost and
    pinned vertices are its fixed set, so its A_free is the owned-free block
    used by the AMG / Jacobi preconditioner) and the qn_slab stage object."""

    def __init__(self, lay: SlabLayout, verts_local, tets_local, material: MaterialModel, pinned_global,
                 h, gravity, density=1000.0, solver="amg", pcg_tol=1e-10, pcg_maxit=20000,
                 fit_interval: FitInterval = FitInterval()):
        import torch

        self.lay = lay
        self.pcg_maxit = int(pcg_maxit)
        n = lay.n
        pin = np.zeros(n, dtype=bool)
        pg = np.asarray(pinned_global, dtype=np.int64)
        pg = pg[(pg >= lay.v0) & (pg < lay.v0 + n)] - lay.v0
        pin[pg] = True
        self.pinned = pin
        owned = np.zeros(n, dtype=bool)
        owned[lay.own_lo:lay.own_hi] = True
        local_fixed = np.nonzero(pin | ~owned)[0]
        mesh = TetMesh(np.ascontiguousarray(verts_local, dtype=np.float64),
                       np.ascontiguousarray(tets_local, dtype=np.int64), density)
        if solver not in ("amg", "pcg"):
            raise DynamicsError(f"slab solver {solver!r}: amg | pcg")
        self.system = _build(mesh, [[(np.arange(mesh.tets.shape[0]), material)]], h, gravity, local_fixed,
                             fit_interval, 1, solver=solver, pcg_tol=pcg_tol, pcg_maxit=pcg_maxit)
        Ar = slab_operator(self.system.L, lumped_masses(mesh), h, pin, owned)
        self.A_of = Ar
        self.owned_free = np.nonzero(owned & ~pin)[0]
        self.coarse = False
        self._a = (_lib.i64(Ar.indptr), _lib.i32(Ar.indices), _lib.f64(Ar.data), np.ascontiguousarray(pin, np.uint8))
        d = _lib.SlabDesc()
        d.local = self.system._h
        d.own_lo, d.own_hi, d.tet_own_lo = lay.own_lo, lay.own_hi, lay.tet_own_lo
        d.pinned = _lib.ptr(self._a[3])
        d.a_nnz = Ar.nnz
        d.a_indptr, d.a_indices, d.a_values = _lib.ptr(self._a[0]), _lib.ptr(self._a[1]), _lib.ptr(self._a[2])
        d.n_ranks, d.pcg_maxit, d.pcg_tol = lay.world, int(pcg_maxit), float(pcg_tol)
        h_ = C.c_void_p()
        _lib.check(_lib.load().qn_slab_create(C.byref(d), C.byref(h_)), "slab_create")
        self._h = h_
        self.buf = {}
        for which in (SEND, GATHER, P, R0, QL, QPREV, Y, X, G):
            p, cnt = C.c_void_p(), C.c_int64()
            _lib.check(_lib.load().qn_slab_buffer(self._h, which, C.byref(p), C.byref(cnt)))
            self.buf[which] = torch.as_tensor(_CudaBuffer(p.value, cnt.value), device="cuda")
        self._args = np.zeros(7 + 2 * RING, dtype=np.float64)

    # -- two-level preconditioner (geometric coarse grid over the whole bar) --
    def coarse_rows(self, cs):
        """P_c rows of every local vertex (CSR, local vertex x coarse node)."""
        lay = self.lay
        return cs.rows(lay.v0 + np.arange(lay.n))

    def coarse_partial(self, cs):
        """This rank's part of A_c = P_c^T A P_c: its owned free rows only, so
        the rank-order sum over slabs is the global Galerkin product (dense)."""
        return galerkin_part(self.A_of, self.coarse_rows(cs), self.owned_free)

    def set_coarse(self, cs, cinv):
        lay = self.lay
        first, w, pos = cs.tables()
        grid = np.asarray(cs.grid, dtype=np.int32)
        dims = np.asarray(cs.dims, dtype=np.int32)
        i_lo = lay.v0 // lay.plane + lay.own_lo // lay.plane
        n_planes = (lay.own_hi - lay.own_lo) // lay.plane
        keep = (grid, dims, first, w, pos, _lib.f64(cinv))
        _lib.check(_lib.load().qn_slab_set_coarse(self._h, _lib.ptr(grid), _lib.ptr(dims), C.c_int64(lay.v0),
                                                  C.c_int64(i_lo), C.c_int64(n_planes), _lib.ptr(first),
                                                  _lib.ptr(w), _lib.ptr(pos), _lib.ptr(keep[5])), "slab_set_coarse")
        self.coarse = True
        self._refresh_buffers((CSEND, CGATHER))

    def _refresh_buffers(self, which):
        import torch
        for w in which:
            p, cnt = C.c_void_p(), C.c_int64()
            _lib.check(_lib.load().qn_slab_buffer(self._h, w, C.byref(p), C.byref(cnt)))
            self.buf[w] = torch.as_tensor(_CudaBuffer(p.value, cnt.value), device="cuda")

    def stage(self, stage, xs=0, xs_to=0, have_prev=0, new_slot=0, ring=(), coef=(), first=0, alpha=0.0):
        import torch
        a = self._args
        a[:] = 0.0
        a[:7] = (xs, xs_to, have_prev, new_slot, len(ring), first, alpha)
        a[7:7 + len(ring)] = ring
        a[7 + RING:7 + RING + len(coef)] = coef
        st = torch.cuda.current_stream().cuda_stream
        _lib.check(_lib.load().qn_slab_stage(self._h, stage, a.ctypes.data, a.size, C.c_void_p(st)), "slab_stage")

    def pcg_status(self):
        import torch
        conv, its = C.c_int32(), C.c_int32()
        st = torch.cuda.current_stream().cuda_stream
        _lib.check(_lib.load().qn_slab_pcg_status(self._h, C.byref(conv), C.byref(its), C.c_void_p(st)))
        return conv.value, its.value

    def plane_slices(self):
        """(ghost lo, own first, own last, ghost hi) element slices of an (n,3) buffer."""
        lay, P3 = self.lay, self.lay.plane * 3
        return (slice(0, P3), slice(lay.own_lo * 3, lay.own_lo * 3 + P3),
                slice(lay.own_hi * 3 - P3, lay.own_hi * 3), slice(lay.n * 3 - P3, lay.n * 3))

    def set_state(self, q_l, q_prev):
        import torch
        for which, a in ((QL, q_l), (QPREV, q_prev)):
            self.buf[which].copy_(torch.as_tensor(np.ascontiguousarray(a, np.float64).reshape(-1)))

    def owned_positions(self):
        lay = self.lay
        return self.buf[QL][lay.own_lo * 3: lay.own_hi * 3].view(-1, 3)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib._lib is not None:
            _lib._lib.qn_slab_destroy(h)
            self._h = None


class EmulatedComm:
    """All ranks' slabs in this process on one device: the all-gather and the
    halo exchange are device copies between their buffers, in rank order,
    on the current stream (no kernel waits on another)."""

    def __init__(self, ranks):
        self.ranks = ranks

    @property
    def local(self):
        return self.ranks

    def allgather(self, pair=(SEND, GATHER)):
        import torch
        allv = torch.cat([rk.buf[pair[0]] for rk in self.ranks])
        for rk in self.ranks:
            rk.buf[pair[1]].copy_(allv)

    def allgather_pair(self, a, b):
        """two all-gathers as one exchange (NcclComm packs them into one collective)"""
        self.allgather(a)
        self.allgather(b)

    def reduce_dense(self, parts):
        """rank-order sum of every rank's dense setup matrix"""
        out = np.zeros_like(parts[0])
        for p in parts:
            out = out + p
        return out

    def same_on_all(self, a):
        return a

    def halo(self, which):
        for lo, hi in zip(self.ranks[:-1], self.ranks[1:]):
            gl, _, last, gh = lo.plane_slices()
            hgl, hfirst, _, _ = hi.plane_slices()
            lo.buf[which][gh].copy_(hi.buf[which][hfirst])
            hi.buf[which][hgl].copy_(lo.buf[which][last])

    def scalars(self):
        return self.ranks[0].buf[GATHER].cpu().numpy().reshape(-1, NSEND)


class NcclComm:
    """One rank per process (torch.distributed, NCCL): all-gather of SEND into
    GATHER and send/recv of the boundary planes with the neighbours."""

    def __init__(self, rank_obj: SlabRank, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rk = rank_obj

    @property
    def local(self):
        return [self.rk]

    def allgather(self, pair=(SEND, GATHER)):
        self.dist.all_gather_into_tensor(self.rk.buf[pair[1]], self.rk.buf[pair[0]], group=self.group)

    def allgather_pair(self, a, b):
        """all-gather of two send buffers in ONE collective: packed [a | b] per rank,
        gathered, unpacked into the two receive buffers (device copies)."""
        import torch
        sa, sb = self.rk.buf[a[0]], self.rk.buf[b[0]]
        na, nb = sa.numel(), sb.numel()
        world = self.dist.get_world_size(self.group)
        if getattr(self, "_pack", None) is None or self._pack[0].numel() != na + nb:
            self._pack = (torch.empty(na + nb, dtype=sa.dtype, device=sa.device),
                          torch.empty(world * (na + nb), dtype=sa.dtype, device=sa.device))
        send, recv = self._pack
        send[:na].copy_(sa)
        send[na:].copy_(sb)
        self.dist.all_gather_into_tensor(recv, send, group=self.group)
        rv = recv.view(world, na + nb)
        self.rk.buf[a[1]].view(world, na).copy_(rv[:, :na])
        self.rk.buf[b[1]].view(world, nb).copy_(rv[:, na:])

    def reduce_dense(self, parts):
        """rank-order sum of every rank's dense setup matrix (all-gather, then
        the same additions on every rank)"""
        import torch
        mine = torch.as_tensor(np.ascontiguousarray(parts[0]), device="cuda")
        world = self.dist.get_world_size(self.group)
        allp = torch.empty((world,) + mine.shape, dtype=mine.dtype, device="cuda")
        self.dist.all_gather_into_tensor(allp, mine, group=self.group)
        allp = allp.cpu().numpy()
        out = np.zeros_like(allp[0])
        for r in range(world):
            out = out + allp[r]
        return out

    def same_on_all(self, a):
        """rank 0's array on every rank (setup results computed redundantly)"""
        import torch
        t = torch.as_tensor(np.ascontiguousarray(a), device="cuda")
        self.dist.broadcast(t, 0, group=self.group)
        return t.cpu().numpy()

    def halo(self, which):
        dist, rk = self.dist, self.rk
        lay = rk.lay
        gl, first, last, gh = rk.plane_slices()
        buf = rk.buf[which]
        ops = []
        if lay.rank > 0:
            ops.append(dist.P2POp(dist.isend, buf[first], lay.rank - 1, group=self.group))
            ops.append(dist.P2POp(dist.irecv, buf[gl], lay.rank - 1, group=self.group))
        if lay.rank < lay.world - 1:
            ops.append(dist.P2POp(dist.isend, buf[last], lay.rank + 1, group=self.group))
            ops.append(dist.P2POp(dist.irecv, buf[gh], lay.rank + 1, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def scalars(self):
        return self.rk.buf[GATHER].cpu().numpy().reshape(-1, NSEND)


class CoarseSpace:
    """Trilinear hat functions on a coarse grid of the bar (index space: coarse
    node I of dimension d sits at fine index min(I f_d, n_d)); the coarse level
    of the slabs' two-level preconditioner.  f_d >= 2 keeps A_c = P^T A P a
    27-point operator."""

    def __init__(self, grid, target=(40, 5, 5)):
        self.grid = tuple(grid)
        self.f = tuple(max(2, -(-n // t)) for n, t in zip(grid, target))
        self.pos = [np.minimum(np.arange(-(-n // f) + 1) * f, n) for n, f in zip(grid, self.f)]
        self.dims = tuple(p.size for p in self.pos)
        self.n = int(np.prod(self.dims))

    def _hat(self, d, i):
        pos = self.pos[d]
        I = np.clip(np.searchsorted(pos, i, side="right") - 1, 0, pos.size - 2)
        t = (i - pos[I]) / (pos[I + 1] - pos[I])
        return I, 1.0 - t, t

    def tables(self):
        """Per-dimension hat tables for the device (x, y, z concatenated): first
        coarse node of each fine index's cell, its two weights, node positions."""
        first, w, pos = [], [], []
        for d, n in enumerate(self.grid):
            I, a0, a1 = self._hat(d, np.arange(n + 1))
            first.append(I.astype(np.int32))
            w.append(np.stack([a0, a1], axis=1).reshape(-1))
            pos.append(self.pos[d].astype(np.int32))
        return np.concatenate(first), np.concatenate(w), np.concatenate(pos)

    def rows(self, gids):
        """P_c rows of global vertex ids (scipy CSR, len(gids) x n)."""
        nx, ny, nz = self.grid
        gids = np.asarray(gids, dtype=np.int64)
        i, rem = np.divmod(gids, (ny + 1) * (nz + 1))
        j, k = np.divmod(rem, nz + 1)
        (Ix, ax0, ax1), (Iy, ay0, ay1), (Iz, az0, az1) = self._hat(0, i), self._hat(1, j), self._hat(2, k)
        Cy, Cz = self.dims[1], self.dims[2]
        rows, cols, vals = [], [], []
        for dx, wx in ((0, ax0), (1, ax1)):
            for dy, wy in ((0, ay0), (1, ay1)):
                for dz, wz in ((0, az0), (1, az1)):
                    w = wx * wy * wz
                    nzm = w != 0.0
                    rows.append(np.nonzero(nzm)[0])
                    cols.append((((Ix + dx) * Cy + (Iy + dy)) * Cz + (Iz + dz))[nzm])
                    vals.append(w[nzm])
        return scipy.sparse.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                       shape=(gids.size, self.n))


def galerkin_part(A_of, P_local, owned_free):
    """P_own^T (A_of P_local), dense: a slab's share of P_c^T A P_c (the rows
    of A_of are the slab's owned free rows; P_local has a row per local vertex)."""
    return (P_local[owned_free].T @ (A_of @ P_local)).toarray()


def setup_coarse(comm, grid, target=(40, 5, 5)):
    """Two-level preconditioner for the slabs of `comm`: every rank's part of
    the Galerkin product, summed in rank order, inverted (rank 0's inverse on
    every rank), and each rank's rows of P_c and P_c^T uploaded."""
    cs = CoarseSpace(grid, target)
    Ac = comm.reduce_dense([rk.coarse_partial(cs) for rk in comm.local])
    Ac = 0.5 * (Ac + Ac.T)
    cinv = comm.same_on_all(np.linalg.inv(Ac))
    for rk in comm.local:
        rk.set_coarse(cs, cinv)
    return cs


def rank_sum(vals):
    """sum over ranks in index order (the device kernels' order)"""
    out = np.zeros(vals.shape[1])
    for r in range(vals.shape[0]):
        out = out + vals[r]
    return out


class SlabRun:
    """simulate_frame (solvers.py:260-352) over the slabs of `comm` (lbfgs with
    lbfgs_init="system_matrix" or pd_qn; no colliders; fixed rows held at q_l)."""

    def __init__(self, comm, config: SolverConfig, h, grad_tol, pcg_check=4):
        if config.kind not in ("lbfgs", "pd_qn"):
            raise NotImplementedError(f"slab frame: solver kind {config.kind!r}")
        if config.m > MAX_M:
            raise SolverError(f"slab frame: m <= {MAX_M}")
        self.comm, self.cfg, self.h = comm, config, float(h)
        self.grad_tol = float(grad_tol)
        self.pcg_check = int(pcg_check)
        self.cg_iterations = 0
        self.last_ms = 0.0

    # -- helpers -------------------------------------------------------------
    def enable_profile(self, on=True):
        """Record CUDA events around every stage / exchange (diagnostics:
        `stage_ms()` sums them per stage after the frame)."""
        self._prof = [] if on else None

    def _ev(self, name, fn):
        if getattr(self, "_prof", None) is None:
            return fn()
        import torch
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        self._prof.append((name, a, b))
        return out

    def stage_ms(self):
        import torch
        torch.cuda.synchronize()
        tot = {}
        for name, a, b in self._prof or []:
            n, t = tot.get(name, (0, 0.0))
            tot[name] = (n + 1, t + a.elapsed_time(b))
        return tot

    def _stage(self, st, **k):
        def go():
            for rk in self.comm.local:
                rk.stage(st, **k)
        self._ev(_STAGE_NAMES[st], go)

    def _gather(self):
        self._ev("allgather", self.comm.allgather)
        return rank_sum(self.comm.scalars())

    def _energy(self, xs):
        self._stage(EVAL, xs=xs)
        v = self._gather()
        return 0.5 / self.h ** 2 * v[1] + v[0]

    def _precondition(self):
        """z = B_slab r (done by the preceding stage) [+ P_c A_c^-1 sum_ranks P_c^T r],
        and the scalars of the next CG step, with ONE collective: the rank's
        <r, r> and <r, B_slab r> partials (SEND) travel with its coarse share
        P_c^T r (CSEND); every rank then forms r_c, e_c = A_c^-1 r_c and the
        coarse term <r_c, e_c> of <r, z> identically (qn_slab.cu k_slab_coarse_dot)."""
        if self.comm.local[0].coarse:
            self._stage(COARSE_R)
            self._stage(PCG_RZ)
            self._ev("allgather", lambda: self.comm.allgather_pair((SEND, GATHER), (CSEND, CGATHER)))
            self._stage(COARSE_APPLY)
        else:
            self._stage(PCG_RZ)
            self._ev("allgather", self.comm.allgather)

    def _solve(self, ring, zeta):
        """r0 = A_free^-1 (-g - sum zeta t) by CG over the slabs (3 columns).
        Collectives per CG iteration: the plane exchange of p, one all-gather
        of <p, q>, one all-gather of <r, r>, <r, z> (+ the coarse shares)."""
        self._stage(PCG_SETUP, ring=ring, coef=zeta)
        self._precondition()
        self._stage(PCG_P, first=1)
        it = 0
        while True:
            self._ev("halo", lambda: self.comm.halo(P))
            self._stage(PCG_SPMV)
            self._ev("allgather", self.comm.allgather)
            self._stage(PCG_UPDATE)
            self._precondition()
            self._stage(PCG_P, first=0)
            it += 1
            if it % self.pcg_check == 0:
                conv, its = self.comm.local[0].pcg_status()
                if conv & 8:
                    self.cg_iterations += its
                    if conv & 7 != 7:  # stopped at pcg_maxit short of pcg_tol
                        raise SolverError("slab frame: PCG stopped at pcg_maxit before reaching pcg_tol")
                    break
                if it > self.comm.local[0].pcg_maxit + self.pcg_check:  # host-side bound on the stage loop
                    raise SolverError("slab frame: PCG did not report convergence within pcg_maxit iterations")
        self._stage(STORE)
        self._ev("halo", lambda: self.comm.halo(R0))

    # -- one frame -------------------------------------------------------------
    def step(self) -> ConvergenceRecord:
        cfg = self.cfg
        lbfgs = cfg.kind == "lbfgs"
        m = cfg.m if lbfgs else 0
        t0 = time.perf_counter()
        rec = ConvergenceRecord()

        def log(g, tr, a):
            rec.g.append(g)
            rec.ls_trials.append(tr)
            rec.alphas.append(a)
            rec.cum_ms.append(1000.0 * (time.perf_counter() - t0))

        self._stage(INIT)
        cur = 0
        g_x = self._energy(cur)
        rec.g0 = g_x
        ring, rho, gram, sg = [], {}, {}, {}
        have_prev = False
        for _ in range(cfg.iterations):
            new_slot = next(s for s in range(RING) if s not in ring)
            self._stage(GRAD, xs=cur, have_prev=int(have_prev and lbfgs), new_slot=new_slot, ring=ring)
            v = self._gather()
            if lbfgs and have_prev:  # LbfgsHistory.push (solvers.py:83-103)
                st, ss, tt = v[1], v[2], v[3]
                if not st <= CURVATURE_GUARD * math.sqrt(ss) * math.sqrt(tt):
                    for j, slot in enumerate(ring):
                        gram[(slot, new_slot)] = v[4 + j]
                    for j, slot in enumerate(ring):
                        sg[slot] = v[4 + MAX_M + j]
                    sg[new_slot] = v[4 + 2 * MAX_M]
                    ring = ring + [new_slot]
                    rho[new_slot] = st
                    if len(ring) > m:
                        ring = ring[1:]
                else:
                    for j, slot in enumerate(ring):
                        sg[slot] = v[4 + MAX_M + j]
            else:
                for j, slot in enumerate(ring):
                    sg[slot] = v[4 + MAX_M + j]
            have_prev = True
            if math.sqrt(v[0]) <= self.grad_tol:  # solvers.py:292-298
                log(g_x, 0, 0.0)
                continue
            # first loop, newest -> oldest: zeta_i = <s_i, q> / rho_i with q = -g - sum_{newer} zeta t
            zeta = {}
            for i in reversed(ring):
                sq = -sg[i]
                for j in ring[ring.index(i) + 1:]:
                    sq -= zeta[j] * gram[(i, j)]
                zeta[i] = sq / rho[i]
            self._solve(ring, [zeta[i] for i in ring])
            coef = []
            if ring:
                self._stage(ETA, ring=ring)
                tr = self._gather()
                cmap = {}
                for k, i in enumerate(ring):  # second loop, oldest -> newest
                    tdot = tr[k]
                    for j in ring[:k]:
                        tdot += cmap[j] * gram[(j, i)]
                    cmap[i] = zeta[i] - tdot / rho[i]
                coef = [cmap[i] for i in ring]
            self._stage(DIR, ring=ring, coef=coef)
            slope = self._gather()[0]
            other = 1 - cur
            if cfg.line_search:
                if slope >= 0.0:
                    raise SolverError(f"line search: ascent direction (slope={slope})")
                if -slope <= 1e-12 * max(abs(g_x), 1.0):  # solvers.py:319-326
                    log(g_x, 0, 0.0)
                    continue
                alpha, trials, accepted = cfg.alpha_init, 0, False
                while True:
                    alpha *= cfg.alpha_shrink
                    if alpha < ALPHA_FLOOR:
                        break
                    trials += 1
                    self._stage(TRIAL, xs=cur, xs_to=other, alpha=alpha)
                    g_new = self._energy(other)
                    if g_new <= g_x + cfg.gamma * alpha * slope:
                        accepted = True
                        break
                if not accepted:  # StagnationError (solvers.py:329-336)
                    rec.stagnated = True
                    while len(rec.g) < cfg.iterations:
                        log(g_x, 0, 0.0)
                    # forces were last evaluated at a rejected trial: not needed (frame ends)
                    break
            else:
                alpha, trials = 1.0, 1
                self._stage(TRIAL, xs=cur, xs_to=other, alpha=1.0)
                g_new = self._energy(other)
            cur = other
            g_x = g_new
            log(g_new, trials, alpha)
        self._stage(FINISH, xs=cur)
        self.last_ms = 1000.0 * (time.perf_counter() - t0)
        return rec


def grad_tolerance(rest_verts_bbox_diag, max_mass, h):
    """grad_tol of solvers.py:278 (scale = rest bounding-box diagonal, dynamics.py:416-417)."""
    return 1e-12 * rest_verts_bbox_diag * max(1.0, max_mass / h ** 2)


def scene_slabs(sc, world, ranks=None, solver="amg", pcg_tol=1e-10, pcg_maxit=20000):
    """SlabRank objects of `ranks` (default: all) for a grid-bar Scene
    (scenes.py; sc.grid set, global arrays), with their initial state."""
    from paper_1604_07378_b200.materials import from_spec
    mat = from_spec(sc.material)
    out = []
    for r in (range(world) if ranks is None else ranks):
        lay = slab_layout(sc.grid, world, r)
        sl = slice(lay.v0, lay.v0 + lay.n)
        rk = SlabRank(lay, sc.verts[sl], local_tets_from_global(sc.tets, lay), mat, sc.fixed, sc.h, sc.gravity,
                      sc.density, solver=solver, pcg_tol=pcg_tol, pcg_maxit=pcg_maxit)
        rk.set_state(sc.q_l[sl], sc.q_prev[sl])
        out.append(rk)
    return out


def scene_grad_tol(sc):
    mesh = TetMesh(sc.verts, sc.tets, sc.density)
    bbox = sc.verts.max(axis=0) - sc.verts.min(axis=0)
    return grad_tolerance(float(np.linalg.norm(bbox)) or 1.0, float(lumped_masses(mesh).max()), sc.h)


def gather_positions(ranks):
    """global (n,3) positions from the owned ranges of emulated ranks"""
    return np.concatenate([rk.owned_positions().cpu().numpy() for rk in ranks])
