"""Batch sharding of the SV hot path across ranks.

The sequence is the unit that shards: rank r of `world` owns the contiguous global sequences
[begin, end) and passes `seq_base = begin` to `sd_verify`, so the Philox counter -- and hence
every output -- is identical to a single-GPU run over the global batch.  There is no data-path
collective; `gather_rows` is only for checking / reporting outside any timed region.
"""
from __future__ import annotations

import torch


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split of `total` sequences: [floor(r*T/W), floor((r+1)*T/W))."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard request")
    return (rank * total) // world, ((rank + 1) * total) // world


def weak_range(per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank owns `per_rank` sequences of a global batch of per_rank*world."""
    return rank * per_rank, (rank + 1) * per_rank


def gather_rows(x: torch.Tensor, total: int, group=None) -> torch.Tensor | None:
    """Gather per-rank row blocks (first dim = this rank's sequences) to rank 0 in global order.
    Works with any torch.distributed backend (gloo on CPU, NCCL on GPU)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(total, world, r)[1] - shard_range(total, world, r)[0] for r in range(world)]
    m = max(sizes)
    pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[: x.shape[0]] = x
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, bufs, dst=0, group=group)
    if rank != 0:
        return None
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)
