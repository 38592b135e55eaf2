"""Pair sharding across ranks.

Stereo pairs are independent, so a multi-GPU job gives every rank its own
contiguous block of pairs and runs the whole matching core locally: no data
exchange, no NCCL on the compute path. The only collective is the
max-over-ranks reduction of the timings (and an optional gather of results for
callers that want them on one rank). torch.distributed is plumbing here:
`nccl` on B200 nodes, `gloo` in the CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int  # first pair (and generator seed offset) of this rank
    count: int


def weak_shard(per_rank: int, rank: int, world: int, seed0: int = 0) -> Shard:
    """Weak scaling: every rank matches `per_rank` pairs, seeds rank*per_rank...
    (BASELINE.json config 2 generator seeds continue across ranks)."""
    if world < 1 or not 0 <= rank < world or per_rank < 0:
        raise ValueError("bad shard request")
    return Shard(rank, world, seed0 + rank * per_rank, per_rank)


def strong_shard(total: int, rank: int, world: int, seed0: int = 0) -> Shard:
    """Strong scaling: `total` pairs split into contiguous blocks
    [r*total/world, (r+1)*total/world)."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard request")
    a = rank * total // world
    b = (rank + 1) * total // world
    return Shard(rank, world, seed0 + a, b - a)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank timing over all ranks (the bench's step time)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() == "gloo":
        device = None  # gloo reduces host tensors
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_rank0(array, device=None):
    """Concatenate equally shaped per-rank numpy arrays on rank 0 (None elsewhere)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return array
    t = torch.from_numpy(np.ascontiguousarray(array))
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    if dist.get_rank() != 0:
        return None
    return np.concatenate([p.cpu().numpy() for p in parts], axis=0)
