"""Data-parallel sharding of independent series over ranks.

Series are independent units: rank r of P gets the contiguous block
[r*B//P, (r+1)*B//P).  There is no exchange step during compute; the only collectives
are after it (gathering sigma / info for reporting), issued by the caller through
torch.distributed.
"""
from __future__ import annotations


def shard_range(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of series owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world) or batch < 0:
        raise ValueError("bad shard request")
    return (rank * batch) // world, ((rank + 1) * batch) // world


def gather_rows(local, world: int, group=None):
    """all_gather of equally- or unequally-sized row blocks (first dim) via padding.
    Works with any torch.distributed backend (nccl on GPU, gloo in CPU tests)."""
    import torch
    import torch.distributed as dist
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)
