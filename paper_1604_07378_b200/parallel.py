"""Multi-GPU decomposition helper for configs[3] (host side).

configs[3] is 1024 independent instances: `shard_instances` splits the
instance range evenly over ranks; every rank builds its own batched system and
no collective touches the data path (bench.py --config c4, strong scaling of a
fixed total).  configs[4] (one large mesh split into x-slabs with halo
exchange and NCCL reductions) lives in `slab.py`.
"""

from __future__ import annotations


def shard_instances(n_inst: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced instance range [lo, hi) of `rank`."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    base, extra = divmod(n_inst, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)
