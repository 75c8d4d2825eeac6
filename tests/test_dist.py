"""Multi-rank host logic on CPU: world_size-2 gloo process group, one library context
per rank (host calls only -- partition, local numbering, halo lists; no device needed).

Checks: labels identical on every rank; owned cells partition the mesh exactly once; the dual-set
partition balances the fine set and the coarse set separately; for every pair of
ranks the send list of one equals the receive list of the other, element by element (global ids),
for the ring-1 exchange, the rings 1-2 exchange and the remote-owned edge exchange.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from inputs.configs import config1, small_shelf


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, which, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2405_10505_b200._abi as abi
        c = config1() if which == "cfg1" else small_shelf(nx=64, ny=48, seed=5)
        ctx = abi.fblts_create(c.dt, c.M, rank=rank, nranks=world)
        abi.fblts_upload_mesh(ctx, c.mesh)
        abi.fblts_set_regions(ctx, c.fine_mask)
        cell, edge = abi.fblts_get_labels(ctx, c.mesh.nCells, c.mesh.nEdges)
        counts = abi.fblts_get_counts(ctx)
        halos = {(x, p): [a.tolist() for a in abi.fblts_get_halo(ctx, x, p)]
                 for x in range(3) for p in range(world) if p != rank}
        abi.fblts_destroy(ctx)
        obj = [None] * world
        dist.all_gather_object(obj, {"cell": cell.tolist(), "edge": edge.tolist(), "counts": counts.tolist(),
                                     "halos": halos})
        if rank == 0:
            q.put(obj)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module", params=["cfg1", "shelf"])
def gathered(request):
    from paper_2405_10505_b200 import build
    build.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, request.param, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = config1() if request.param == "cfg1" else small_shelf(nx=64, ny=48, seed=5)
    return c, out


def test_labels_identical_on_every_rank(gathered):
    _, out = gathered
    assert out[0]["cell"] == out[1]["cell"] and out[0]["edge"] == out[1]["edge"]


def test_owned_cells_partition_the_mesh(gathered):
    c, out = gathered
    owned = [o["counts"][21] for o in out]
    assert sum(owned) == c.mesh.nCells and all(n > 0 for n in owned)
    # dual-set balance: each rank owns half of the fine set and half of the coarse set (+-1)
    fine = [sum(o["counts"][3 + 3:3 + 9]) for o in out]          # owned cells with region code >= 3
    nfine = int(np.count_nonzero(c.fine_mask))
    assert sum(fine) == nfine and max(fine) - min(fine) <= 1
    coarse = [owned[r] - fine[r] for r in range(2)]
    assert max(coarse) - min(coarse) <= 1


@pytest.mark.parametrize("which", [0, 1, 2])
def test_send_lists_match_receive_lists(gathered, which):
    _, out = gathered
    s01, r01 = out[0]["halos"][(which, 1)]
    s10, r10 = out[1]["halos"][(which, 0)]
    assert s01 == r10 and s10 == r01
    assert len(s01) > 0 and len(s10) > 0
    assert s01 == sorted(s01) and len(set(s01)) == len(s01)
