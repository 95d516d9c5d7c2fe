"""Sharding across the GPUs of one box (one process per GPU).

Batch sharding (configs c3 at 1/2/4/8 GPUs):

Requests are independent (Alg. 2, "foreach draft t in T in parallel"), so the data
path has no collective: rank r verifies its own requests, identified by GLOBAL request ids
(Philox is keyed by them, reading #8, so results do not depend on the sharding).
The process group is used only to time the step as the max over ranks and to aggregate the
verified-token count (plumbing, not the product path).

Vocabulary sharding (config c5): every rank holds a contiguous column shard of
every row; the library's own NCCL communicator carries the three small exchanges inside
cosine_verify_batch.  `vocab_shard` gives the shard, `init_vocab_sharded` the collective init
(rank 0 makes the NCCL unique id; the bytes are broadcast over the torch process group).
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


def vocab_shard(V: int, world: int, rank: int, align: int = 8) -> tuple[int, int]:
    """Contiguous column shard [begin, end) of a V-wide vocabulary for `rank`; shards tile
    [0, V) in rank order.  Boundaries are rounded to `align` columns where V allows it."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    def edge(r):
        if r == 0:
            return 0
        if r == world:
            return V
        return min(V, (V * r // world + align // 2) // align * align)
    b, e = edge(rank), edge(rank + 1)
    if e <= b:
        raise ValueError(f"vocabulary of {V} too narrow for {world} shards")
    return b, e


def init_vocab_sharded(V: int, *, device: int, max_batch: int, max_draft_len: int, max_drafters: int,
                       world: int | None = None, rank: int | None = None, **kw):
    """Collective init of a vocabulary-sharded context over the torch process group's ranks."""
    import torch.distributed as dist
    from ._lib import cosine_nccl_unique_id, cosine_verify_init
    world = dist.get_world_size() if world is None else world
    rank = dist.get_rank() if rank is None else rank
    obj = [cosine_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    b, e = vocab_shard(V, world, rank)
    return cosine_verify_init(V, device=device, max_batch=max_batch, max_draft_len=max_draft_len,
                              max_drafters=max_drafters, nranks=world, rank=rank, vocab_begin=b,
                              vocab_end=e, nccl_unique_id=obj[0], **kw)
