"""Distributed set-up for weak scaling (reading Q25; fblts_set_partition) on CPU: a
world_size-2 gloo group in which each rank generates ONLY its piece of the weak-scaled config-5
recipe (inputs.configs.config5_weak_piece: its block of rows plus a margin of its neighbours' rows),
labels it and builds its halo lists locally.  Checked against the single-process set-up of the whole
mesh (the block stacked twice in y, uploaded whole with the same row-block partition):

* labels of every owned and halo cell equal the whole mesh's labels at the same global cell;
* owned cells partition the whole mesh exactly once;
* every halo list (ring-1 cells, rings 1-2 cells, remote-owned edges) equals the whole-mesh set-up's
  list element by element, in whole-mesh ids, and rank r's send list to p equals p's receive list
  from r (the two sides of each exchange agree without having seen each other's piece).
Host logic only (no device)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from inputs import configs
from inputs.hexmesh import build_periodic_hex_mesh_fast

NX, NY, WORLD = 48, 48, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def setup_lists(abi, mesh, fine, owner, gid, rank, world, dt):
    ctx = abi.fblts_create(dt, 4, rank=rank, nranks=world)
    abi.fblts_upload_mesh(ctx, mesh)
    abi.fblts_set_partition(ctx, owner, gid)
    abi.fblts_set_regions(ctx, fine)
    cell, _ = abi.fblts_get_labels(ctx, mesh.nCells, mesh.nEdges)
    counts = abi.fblts_get_counts(ctx)
    halos = {(x, p): [a.tolist() for a in abi.fblts_get_halo(ctx, x, p)]
             for x in range(3) for p in range(world) if p != rank}
    abi.fblts_destroy(ctx)
    return cell, counts, halos


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2405_10505_b200._abi as abi
        pc = configs.config5_weak_piece(rank, world, nx=NX, ny=NY)
        c = pc.case
        cell, counts, halos = setup_lists(abi, c.mesh, c.fine_mask, pc.owner, pc.gid, rank, world, c.dt)
        own_gid = pc.gid[pc.own].tolist()
        # labels by whole-mesh id for the cells this rank holds (owned + the two halo rings)
        held = sorted(set(own_gid) | {g for (x, p), (snd, rcv) in halos.items() if x == 1 for g in rcv})
        g2p = {int(g): k for k, g in enumerate(pc.gid)}
        labels = {g: int(cell[g2p[g]]) for g in held}
        obj = [None] * world
        dist.all_gather_object(obj, {"own": own_gid, "halos": halos, "labels": labels, "nown": int(counts[21])})
        if rank == 0:
            q.put(obj)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def pieces_and_whole():
    from paper_2405_10505_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the whole weak mesh in one process: the block stacked WORLD times, same row-block owners
    import paper_2405_10505_b200._abi as abi
    blk = configs.config5_weak_piece(0, 1, nx=NX, ny=NY).case
    mesh = build_periodic_hex_mesh_fast(NX, NY * WORLD, 500.0)
    j, i = np.divmod(np.arange(mesh.nCells), NX)
    bcell = (j % NY) * NX + i
    mesh.bottomDepth = blk.mesh.bottomDepth[bcell]
    mesh.fVertex = np.full(mesh.nVertices, configs.F_PLANE)
    owner = (j // NY).astype(np.int32)
    gid = np.arange(mesh.nCells, dtype=np.int64)
    whole = [setup_lists(abi, mesh, blk.fine_mask[bcell], owner, gid, r, WORLD, blk.dt) for r in range(WORLD)]
    return out, whole, mesh


def test_owned_cells_partition_the_whole_mesh(pieces_and_whole):
    out, _, mesh = pieces_and_whole
    owned = sorted(g for o in out for g in o["own"])
    assert owned == list(range(mesh.nCells))
    assert all(o["nown"] == NX * NY for o in out)


def test_piece_labels_equal_whole_mesh_labels(pieces_and_whole):
    out, whole, _ = pieces_and_whole
    for r, o in enumerate(out):
        cell_whole = whole[r][0]
        bad = [g for g, lab in o["labels"].items() if cell_whole[g] != lab]
        assert not bad, (r, bad[:5])


def test_piece_halo_lists_equal_whole_mesh_lists(pieces_and_whole):
    out, whole, _ = pieces_and_whole
    for r, o in enumerate(out):
        for key, (snd, rcv) in o["halos"].items():
            wsnd, wrcv = whole[r][2][key]
            assert snd == wsnd and rcv == wrcv, (r, key)
            assert len(snd) > 0


def test_piece_exchanges_agree_pairwise(pieces_and_whole):
    out, _, _ = pieces_and_whole
    for r in range(WORLD):
        for p in range(WORLD):
            if p == r:
                continue
            for x in range(3):
                assert out[r]["halos"][(x, p)][0] == out[p]["halos"][(x, r)][1], (r, p, x)
