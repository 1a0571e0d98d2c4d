"""Multi-GPU decomposition helpers (host side, torch.distributed for the plumbing).

* configs[3] (independent instances): `shard_instances` splits the instance
  range evenly over ranks; every rank builds its own batched system and no
  collective touches the data path (bench.py --config c4).
* configs[4] (one large mesh): `slab_partition` assigns grid cells to ranks as
  slabs along x and derives each rank's tets, owned vertices and the
  one-vertex-plane halo shared with each neighbour; `halo_sum` adds the
  partial interface contributions of the neighbouring slabs (fixed order:
  lower rank first, so the sum is deterministic and identical on both
  sides); `allreduce_sum` reduces scalars (dots, energies) across ranks.
  These primitives are exercised with world_size 2 over gloo in
  tests/test_parallel.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_instances(n_inst: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced instance range [lo, hi) of `rank`."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    base, extra = divmod(n_inst, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class Slab:
    rank: int
    cells: tuple          # [i0, i1) cell range along x
    tets: np.ndarray      # global tet ids of the slab (Freudenthal order)
    verts: np.ndarray     # global vertex ids touched by the slab (sorted)
    halo_lo: np.ndarray   # global ids of the plane shared with rank - 1 (or empty)
    halo_hi: np.ndarray   # global ids of the plane shared with rank + 1 (or empty)


def slab_partition(grid, world: int, rank: int) -> Slab:
    """Slab of a Freudenthal bar (vertex id (i(ny+1)+j)(nz+1)+k, 6 tets per
    cell in C order, as mesh.grid_bar) for `rank` of `world`."""
    nx, ny, nz = grid
    lo, hi = shard_instances(nx, world, rank)
    per_cell = 6 * ny * nz
    tets = np.arange(lo * per_cell, hi * per_cell, dtype=np.int64)
    plane = (ny + 1) * (nz + 1)
    verts = np.arange(lo * plane, (hi + 1) * plane, dtype=np.int64)
    halo_lo = np.arange(lo * plane, (lo + 1) * plane, dtype=np.int64) if rank > 0 else np.zeros(0, np.int64)
    halo_hi = np.arange(hi * plane, (hi + 1) * plane, dtype=np.int64) if rank < world - 1 else np.zeros(0, np.int64)
    return Slab(rank, (lo, hi), tets, verts, halo_lo, halo_hi)


def halo_sum(local, slab: Slab, dist, group=None):
    """Sum the partial (n_local, 3) contributions on the shared planes with the
    neighbouring slabs.  `local` is indexed by `slab.verts`; returns a new
    tensor.  The shared rows become (lower rank's part) + (upper rank's part)
    on both ranks."""
    import torch
    out = local.clone()
    world = dist.get_world_size(group)
    base = slab.verts[0]
    reqs, bufs = [], {}
    for side, halo, peer in (("lo", slab.halo_lo, slab.rank - 1), ("hi", slab.halo_hi, slab.rank + 1)):
        if halo.size == 0 or not (0 <= peer < world):
            continue
        idx = torch.as_tensor(halo - base, device=local.device)
        send = local.index_select(0, idx).contiguous()
        recv = torch.empty_like(send)
        reqs.append(dist.isend(send, peer, group=group))
        reqs.append(dist.irecv(recv, peer, group=group))
        bufs[side] = (idx, send, recv)
    for r in reqs:
        r.wait()
    for side, (idx, send, recv) in bufs.items():
        lower_first = (recv + send) if side == "lo" else (send + recv)
        out.index_copy_(0, idx, lower_first)
    return out


def allreduce_sum(values, dist, group=None):
    """Sum a small float64 tensor of scalars over ranks (in place)."""
    dist.all_reduce(values, op=dist.ReduceOp.SUM, group=group)
    return values
