"""Multi-GPU plumbing for the render path.

The path shards without any data-path collective:

* C3 (many views): contiguous blocks of views per rank (`shard_views`), the
  scene replicated on every GPU; each rank renders its own views.
* C4 (one large view): pixels are independent; tiles are dealt round-robin
  (`shard_tiles`) so the centred object is balanced across ranks.
* C5 (fitting): each rank runs fwd+bwd for its views, then ONE all-reduce(sum)
  of the per-kernel gradients (`allreduce_gradients`) — the only collective,
  NCCL over NVLink on GPUs (gloo in the CPU tests).

One process per GPU; torch.distributed provides the process group.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np


def shard_views(n_views: int, rank: int, world: int) -> List[int]:
    """Contiguous block of view indices for `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return list(range(start, start + count))


def shard_tiles(n_tiles: int, rank: int, world: int) -> np.ndarray:
    """Round-robin tile ids for `rank` (balances a centred object)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    return np.arange(rank, n_tiles, world, dtype=np.int64)


def allreduce_gradients(tensors: Sequence, group=None) -> None:
    """Sum per-kernel gradient tensors (torch) across ranks in place.

    The tensors are flattened into one contiguous buffer so a single collective
    is issued per iteration (bucket = the whole gradient, ~1.2-3 MB at 50k
    kernels: launch latency, not bandwidth, dominates on NVLink)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    flat = torch.cat([t.reshape(-1) for t in tensors])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    off = 0
    for t in tensors:
        n = t.numel()
        t.copy_(flat[off:off + n].view_as(t))
        off += n
