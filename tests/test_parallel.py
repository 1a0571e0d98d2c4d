"""Multi-rank host logic on CPU (gloo, world_size 2-4): instance sharding for
configs[3] and the configs[4] slab decomposition (paper_1604_07378_b200/slab.py):
vertex ownership and ghost layers, operator rows, the communicator's
all-gather and plane exchange, and the coarse-space Galerkin parts."""
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


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


# ---- slab decomposition of the configs[4] frame (paper_1604_07378_b200/slab.py) ----

@pytest.mark.parametrize("grid,world", [((7, 2, 2), 1), ((7, 2, 2), 2), ((7, 2, 2), 3), ((9, 3, 2), 4), ((4, 1, 1), 4)])
def test_slab_layout_owns_every_vertex_once_and_sees_all_incident_tets(grid, world):
    from paper_1604_07378_b200 import slab
    verts, tets = O.grid_bar(*grid, (0.1 * grid[0], 0.1 * grid[1], 0.1 * grid[2]))
    n = verts.shape[0]
    owner = np.zeros(n, dtype=int)
    tet_owner = np.zeros(tets.shape[0], dtype=int)
    for r in range(world):
        lay = slab.slab_layout(grid, world, r)
        loc = slab.local_tets_from_global(tets, lay)
        assert np.array_equal(loc, slab.local_tets_generated(lay, (0.1 * grid[0], 0.1 * grid[1], 0.1 * grid[2])))
        assert loc.min() >= 0 and loc.max() < lay.n
        gids = np.arange(lay.own_lo, lay.own_hi) + lay.v0
        owner[gids] += 1
        per = lay.tets_per_cell
        tet_owner[lay.c0 * per: lay.c1 * per] += 1
        # every tet touching an owned vertex is local
        owned = np.zeros(n, dtype=bool)
        owned[gids] = True
        touching = np.nonzero(owned[tets].any(axis=1))[0]
        assert touching.min() >= lay.cl * per and touching.max() < lay.c1 * per
        # ghost planes: one plane below (r > 0) and one above (r < world - 1)
        assert lay.own_lo == (lay.plane if r > 0 else 0)
        assert lay.n - lay.own_hi == (lay.plane if r < world - 1 else 0)
    assert np.all(owner == 1) and np.all(tet_owner == 1)


def test_slab_operator_rows_are_global_A_rows():
    from paper_1604_07378_b200 import slab
    from paper_1604_07378_b200.mesh import TetMesh, lumped_masses, tet_diff_operators
    sc = scenes.c5(grid=(9, 2, 3), frames=1)
    h, k = sc.h, 2.5e6
    mesh = TetMesh(sc.verts, sc.tets, sc.density)
    _, vols = tet_diff_operators(mesh)
    pin_g = np.zeros(mesh.n, dtype=bool)
    pin_g[sc.fixed] = True
    Ag = slab.slab_operator(slab.stiffness_matrix(mesh, vols * k), lumped_masses(mesh), h, pin_g,
                            np.ones(mesh.n, dtype=bool)).toarray()
    free_g = np.nonzero(~pin_g)[0]
    row_of = {v: i for i, v in enumerate(free_g)}
    for world in (2, 3):
        for r in range(world):
            lay = slab.slab_layout(sc.grid, world, r)
            lm = TetMesh(sc.verts[lay.v0: lay.v0 + lay.n], slab.local_tets_from_global(sc.tets, lay), sc.density)
            _, lv = tet_diff_operators(lm)
            pin = pin_g[lay.v0: lay.v0 + lay.n]
            owned = np.zeros(lay.n, dtype=bool)
            owned[lay.own_lo: lay.own_hi] = True
            Al = slab.slab_operator(slab.stiffness_matrix(lm, lv * k), lumped_masses(lm), h, pin, owned).toarray()
            rows = np.nonzero(owned & ~pin)[0]
            assert Al.shape[0] == rows.size
            for i, v in enumerate(rows):
                np.testing.assert_allclose(Al[i], Ag[row_of[v + lay.v0], lay.v0: lay.v0 + lay.n], rtol=1e-13,
                                           atol=1e-9)
                # nothing of the global row lies outside the slab
                outside = np.delete(Ag[row_of[v + lay.v0]], np.arange(lay.v0, lay.v0 + lay.n))
                assert not outside.any()


class _StubRank:
    """CPU stand-in with a SlabRank's buffers and layout (communicator test)."""

    def __init__(self, lay):
        from paper_1604_07378_b200 import slab
        self.lay = lay
        self.buf = {slab.SEND: torch.zeros(slab.NSEND, dtype=torch.float64),
                    slab.GATHER: torch.zeros(lay.world * slab.NSEND, dtype=torch.float64),
                    slab.P: torch.zeros(lay.n * 3, dtype=torch.float64),
                    slab.CSEND: torch.zeros(3 * 7, dtype=torch.float64),
                    slab.CGATHER: torch.zeros(lay.world * 3 * 7, dtype=torch.float64)}

    def plane_slices(self):
        from paper_1604_07378_b200.slab import SlabRank
        return SlabRank.plane_slices(self)


def _comm_worker(rank, world, port, out):
    from paper_1604_07378_b200 import slab
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = slab.slab_layout((6, 2, 1), world, rank)
        rk = _StubRank(lay)
        rk.buf[slab.SEND][:] = torch.arange(slab.NSEND, dtype=torch.float64) + 100 * rank
        gid = torch.arange(lay.n * 3, dtype=torch.float64) + lay.v0 * 3
        rk.buf[slab.P][:] = -1.0
        rk.buf[slab.P][lay.own_lo * 3: lay.own_hi * 3] = gid[lay.own_lo * 3: lay.own_hi * 3]
        comm = slab.NcclComm(rk)
        comm.allgather()
        comm.halo(slab.P)
        gath1 = rk.buf[slab.GATHER].numpy().copy()
        # the CG's merged exchange: scalars and coarse shares in one collective
        rk.buf[slab.SEND][:] = -torch.arange(slab.NSEND, dtype=torch.float64) - 1000 * rank
        rk.buf[slab.CSEND][:] = torch.arange(21, dtype=torch.float64) + 10000 * rank
        comm.allgather_pair((slab.SEND, slab.GATHER), (slab.CSEND, slab.CGATHER))
        out[rank] = (lay, gath1, rk.buf[slab.P].numpy().copy(), gid.numpy(), rk.buf[slab.GATHER].numpy().copy(),
                     rk.buf[slab.CGATHER].numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_communicator_allgather_and_halo(world):
    """NcclComm's all-gather, the CG's merged all-gather of the scalars and the
    coarse shares, and the plane exchange (gloo on CPU): every rank gets every
    SEND (and CSEND) in rank order, and every local vertex (ghost planes
    included) holds its owner's value after the halo exchange."""
    from paper_1604_07378_b200 import slab
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_comm_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    expect = np.concatenate([np.arange(slab.NSEND) + 100.0 * r for r in range(world)])
    exp2 = np.concatenate([-np.arange(slab.NSEND) - 1000.0 * r for r in range(world)])
    exp3 = np.concatenate([np.arange(21) + 10000.0 * r for r in range(world)])
    for r in range(world):
        lay, gath, p, gid, g2, cg2 = out[r]
        np.testing.assert_array_equal(gath, expect)
        np.testing.assert_array_equal(p, gid)
        np.testing.assert_array_equal(g2, exp2)  # allgather_pair: both buffers, rank order
        np.testing.assert_array_equal(cg2, exp3)
    assert np.array_equal(slab.rank_sum(expect.reshape(world, -1)), sum(expect.reshape(world, -1)[r] for r in range(world)))


def test_slab_coarse_space_galerkin_parts_sum_to_global():
    """The two-level preconditioner's coarse operator: the rank-order sum of the
    slabs' Galerkin parts P_own^T A_of P_local is the global P^T A_free P."""
    from paper_1604_07378_b200 import slab
    from paper_1604_07378_b200.mesh import TetMesh, lumped_masses, tet_diff_operators
    sc = scenes.c5(grid=(12, 3, 4), frames=1)
    h, k = sc.h, 2.5e6
    mesh = TetMesh(sc.verts, sc.tets, sc.density)
    _, vols = tet_diff_operators(mesh)
    cs = slab.CoarseSpace(sc.grid, target=(4, 2, 2))
    P = cs.rows(np.arange(mesh.n))
    assert np.allclose(np.asarray(P.sum(axis=1)).ravel(), 1.0)  # partition of unity
    pin_g = np.zeros(mesh.n, dtype=bool)
    pin_g[sc.fixed] = True
    Ag = slab.slab_operator(slab.stiffness_matrix(mesh, vols * k), lumped_masses(mesh), h, pin_g,
                            np.ones(mesh.n, dtype=bool))
    free = np.nonzero(~pin_g)[0]
    ref = slab.galerkin_part(Ag, P, free)
    for world in (2, 3):
        tot = np.zeros_like(ref)
        for r in range(world):
            lay = slab.slab_layout(sc.grid, world, r)
            lm = TetMesh(sc.verts[lay.v0: lay.v0 + lay.n], slab.local_tets_from_global(sc.tets, lay), sc.density)
            _, lv = tet_diff_operators(lm)
            pin = pin_g[lay.v0: lay.v0 + lay.n]
            owned = np.zeros(lay.n, dtype=bool)
            owned[lay.own_lo: lay.own_hi] = True
            Al = slab.slab_operator(slab.stiffness_matrix(lm, lv * k), lumped_masses(lm), h, pin, owned)
            tot = tot + slab.galerkin_part(Al, cs.rows(lay.v0 + np.arange(lay.n)), np.nonzero(owned & ~pin)[0])
        np.testing.assert_allclose(tot, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    assert np.allclose(ref, ref.T, rtol=1e-12, atol=1e-9 * np.abs(ref).max())
