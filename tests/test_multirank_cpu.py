"""World-size-2 gloo run of the batch-sharded path's host logic on CPU: the shards cover the
batch, the step time is the max over ranks, and the union of the ranks' results equals the
unsharded result bit for bit (Philox keyed by global request ids, reading #8).  The per-rank
verification here is the oracle (test infrastructure); on the GPU box the same harness runs the
CUDA path (bench.py --gpus N)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_2503_10325_b200 import sharding
    inp = synth.linear_inputs(10, 4, 3, 300, dtype=torch.float32, seed=3, sigma=3.0)
    b0, b1 = sharding.shard_range(10, world, rank)
    r = oracle.verify_batch(inp["target"][b0:b1], inp["draft"][b0:b1], inp["draft_tokens"][b0:b1],
                            inp["request_ids"][b0:b1], seed=11, vocab=300)
    t = sharding.max_over_ranks(1.0 + rank)
    n = sharding.sum_over_ranks(b1 - b0)
    outs = [None] * world
    dist.all_gather_object(outs, (b0, b1, r["out_tokens"].tolist(), r["accept_len"].tolist()))
    if rank == 0:
        q.put((t, n, outs))
    dist.destroy_process_group()


def test_two_rank_batch_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, n, outs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0 and n == 10
    import oracle
    import synth
    inp = synth.linear_inputs(10, 4, 3, 300, dtype=torch.float32, seed=3, sigma=3.0)
    full = oracle.verify_batch(inp["target"], inp["draft"], inp["draft_tokens"], inp["request_ids"], seed=11,
                               vocab=300)
    merged = np.concatenate([np.array(o[2]) for o in sorted(outs)])
    np.testing.assert_array_equal(merged, full["out_tokens"])
    assert [o[:2] for o in sorted(outs)] == [(0, 5), (5, 10)]


def test_shard_ranges():
    from paper_2503_10325_b200 import sharding
    for total in (1, 7, 256, 1024):
        for world in (1, 2, 4, 8):
            rs = [sharding.shard_range(total, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(e - s for s, e in rs) - min(e - s for s, e in rs) <= 1
    assert list(sharding.weak_request_ids(4, 2)) == [8, 9, 10, 11]
    with pytest.raises(ValueError):
        sharding.shard_range(4, 2, 2)


def _vocab_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_10325_b200 import sharding
    # the unique-id broadcast of init_vocab_sharded, with a stand-in id (no NCCL on CPU)
    obj = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    shards = [sharding.vocab_shard(128256, world, r) for r in range(world)]
    if rank == 0:
        q.put((obj[0], shards))
    else:
        q.put((obj[0], None))
    dist.destroy_process_group()


def test_two_rank_vocab_shard_plumbing():
    """Host logic of the vocabulary-sharded mode: both ranks receive rank 0's id bytes, and the
    column shards tile [0, V) in rank order (c5: 8 x 16032)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vocab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(g[0] == bytes(range(128)) for g in got)
    shards = [g[1] for g in got if g[1] is not None][0]
    assert shards == [(0, 64128), (64128, 128256)]
    from paper_2503_10325_b200 import sharding
    for V, G in [(128256, 8), (5003, 3), (32000, 4), (17, 2)]:
        sh = [sharding.vocab_shard(V, G, r) for r in range(G)]
        assert sh[0][0] == 0 and sh[-1][1] == V
        assert all(sh[r][1] == sh[r + 1][0] and sh[r][0] < sh[r][1] for r in range(G - 1))
    assert [sharding.vocab_shard(128256, 8, r)[1] - sharding.vocab_shard(128256, 8, r)[0] for r in range(8)] == [16032] * 8
