"""Host-side plumbing of the slab decomposition: who owns which
cell planes, and the exchange of the ranks' IPC handles over
torch.distributed. No arithmetic of the method; the exchange itself runs in
libdem's kernels over peer memory."""
from __future__ import annotations


def plane_range(rank: int, world: int, nz: int) -> tuple[int, int]:
    """[z0, z1) of global cell planes owned by `rank` (the library's partition:
    z0 = floor(r nz / P))."""
    return rank * nz // world, (rank + 1) * nz // world


def neighbour_handles(rank: int, world: int, mine: bytes, group=None):
    """All-gather every rank's exchange handle; return (left, right) handles,
    None at the domain ends."""
    import torch.distributed as dist
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    assert allh[rank] == mine
    left = allh[rank - 1] if rank > 0 else None
    right = allh[rank + 1] if rank < world - 1 else None
    return left, right
