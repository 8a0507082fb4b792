"""Multi-GPU plumbing: request sharding and the statistics all-reduce (north_star: trees are
independent, so batches shard by request; NCCL over NVLink only all-reduces aggregates)."""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(rank: int, world: int, trees_per_rank: int, total: int | None = None):
    """Tree ids of this rank: weak scaling gives each rank its own `trees_per_rank` block;
    with `total` set (strong scaling) the ids [0, total) are split as evenly as possible."""
    if total is None:
        return rank * trees_per_rank, trees_per_rank
    lo = (rank * total) // world
    hi = ((rank + 1) * total) // world
    return lo, hi - lo


def allreduce_stats(stats: torch.Tensor, dstats: torch.Tensor, group=None):
    """Sum the int64 A9 statistics vector and the fp64 (Σe_hat, Σutility) pair over ranks."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(dstats, op=dist.ReduceOp.SUM, group=group)
    return stats, dstats


def max_over_ranks(values: torch.Tensor, group=None):
    """Element-wise max over ranks (timings are reported as the slowest rank)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(values, op=dist.ReduceOp.MAX, group=group)
    return values
