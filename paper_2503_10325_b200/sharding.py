"""Batch sharding across the GPUs of one box (one process per GPU).

Requests are independent (Alg. 2, "foreach draft t in T in parallel"), so the data
path has no collective: rank r verifies its own requests, identified by GLOBAL request ids
(Philox is keyed by them, reading #8, so results do not depend on the sharding).
The process group is used only to time the step as the max over ranks and to aggregate the
verified-token count (plumbing, not the product path).
"""
from __future__ import annotations


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) slice of n_total requests owned by `rank` (balanced to +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    return n_total * rank // world, n_total * (rank + 1) // world


def weak_request_ids(batch_per_rank: int, rank: int):
    """Global ids of rank `rank`'s batch under weak scaling (every rank a full batch)."""
    return range(rank * batch_per_rank, (rank + 1) * batch_per_rank)


def max_over_ranks(value: float, device=None) -> float:
    """Step time of a multi-rank run = the slowest rank (all_reduce MAX); identity if N = 1."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
