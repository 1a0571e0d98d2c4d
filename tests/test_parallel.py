"""Multi-rank host logic on CPU (gloo, world_size 2): instance sharding for
configs[3] and the slab decomposition / halo sum / allreduce used by the
configs[4] domain decomposition — the distributed gradient of a slab-split
bar must equal the single-process gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle.qnsim_oracle as O
from paper_1604_07378_b200 import parallel, scenes
from tests.helpers import oracle_material


def test_shard_instances_cover_and_balance():
    for n, w in ((1024, 1), (1024, 2), (1024, 8), (10, 3), (3, 4)):
        spans = [parallel.shard_instances(n, w, r) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        sizes = [hi - lo for lo, hi in spans]
        assert max(sizes) - min(sizes) <= 1


def test_slab_partition_covers_tets_once():
    grid = (12, 3, 2)
    verts, tets = O.grid_bar(*grid, (1.2, 0.3, 0.2))
    seen = np.zeros(tets.shape[0], dtype=int)
    for r in range(3):
        s = parallel.slab_partition(grid, 3, r)
        seen[s.tets] += 1
        assert set(np.unique(tets[s.tets])) <= set(s.verts)  # slab tets only touch slab vertices
        if r > 0:
            assert s.halo_lo.size == 4 * 3
    assert np.all(seen == 1)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = scenes.c1(grid=(8, 2, 2))
        mat = oracle_material(sc.material)
        G, vols = O.diff_operators(sc.verts, sc.tets)
        rng = np.random.default_rng(5)
        x = sc.verts + 0.01 * rng.standard_normal(sc.verts.shape)
        slab = parallel.slab_partition((8, 2, 2), world, rank)
        grp = O.TetGroup(sc.tets[slab.tets], G[slab.tets], vols[slab.tets], mat, 1.0)
        full = np.zeros_like(x)
        grp.add_gradient(x, full)
        local = torch.from_numpy(full[slab.verts].copy())
        summed = parallel.halo_sum(local, slab, dist)
        e = torch.tensor([grp.energy(x)], dtype=torch.float64)
        parallel.allreduce_sum(e, dist)
        out[rank] = (slab.verts, summed.numpy(), float(e[0]))
    finally:
        dist.destroy_process_group()


def test_distributed_gradient_equals_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    sc = scenes.c1(grid=(8, 2, 2))
    mat = oracle_material(sc.material)
    G, vols = O.diff_operators(sc.verts, sc.tets)
    rng = np.random.default_rng(5)
    x = sc.verts + 0.01 * rng.standard_normal(sc.verts.shape)
    grp = O.TetGroup(sc.tets, G, vols, mat, 1.0)
    ref = np.zeros_like(x)
    grp.add_gradient(x, ref)
    e_ref = grp.energy(x)
    for r in range(world):
        verts, g, e = out[r]
        np.testing.assert_allclose(g, ref[verts], rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        assert e == pytest.approx(e_ref, rel=1e-12)
