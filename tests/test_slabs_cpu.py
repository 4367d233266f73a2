"""CPU tests of the slab plumbing (world_size 2 and 3 over gloo): the plane
partition covers every plane exactly once with >= 2 planes per rank, and the
IPC-handle exchange hands each rank exactly its neighbours' handles."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_1301_1714_b200.slabs import neighbour_handles, plane_range


@pytest.mark.parametrize("nz,world", [(23, 2), (23, 3), (261, 8), (97, 4), (16, 8)])
def test_plane_partition(nz, world):
    ranges = [plane_range(r, world, nz) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == nz
    for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
        assert a1 == b0
    assert all(z1 - z0 >= 2 for z0, z1 in ranges)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = bytes([rank]) * 64  # stands in for a cudaIpcMemHandle_t
    left, right = neighbour_handles(rank, world, mine)
    out.put((rank, left, right))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_neighbour_handle_exchange_gloo(world):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (lft, rgt)) for r, lft, rgt in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        lft, rgt = got[r]
        assert lft == (bytes([r - 1]) * 64 if r > 0 else None)
        assert rgt == (bytes([r + 1]) * 64 if r < world - 1 else None)
