"""Vocabulary-sharded parity check (SURVEY §8(e), config c5 layout), one process per GPU:

    torchrun --nproc-per-node G --master-addr 127.0.0.1 tools/shard_check.py [--out F]

Every rank builds the same seeded inputs, keeps its column shard of every row and calls
cosine_verify_batch collectively on a vocabulary-sharded context.  Rank 0 compares the
(replicated) outputs with (a) the unsharded library call on the full rows and (b) the oracle:
accept_len / out_tokens / status bit-exact except flagged near-ties, debug probabilities within
1e-5.  Test infrastructure (imports the oracle); used by tests/test_gpu_vocab_shard.py.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2503_10325_b200 as cv  # noqa: E402
import synth  # noqa: E402
from paper_2503_10325_b200.sharding import vocab_shard  # noqa: E402


def column_shard(x: torch.Tensor, b: int, e: int, pad=float("nan")) -> torch.Tensor:
    """Columns [b, e) of the last dim into a fresh 16-byte-aligned buffer (ld = round_up(e-b, 8))."""
    w = e - b
    ld = (w + 7) // 8 * 8
    out = torch.full(x.shape[:-1] + (ld,), pad, dtype=x.dtype, device=x.device)
    out[..., :w] = x[..., b:e]
    return out


CASES = [
    # name, B, k, N, V, dtype, kwargs
    ("conf_bf16", 24, 6, 3, 5003, torch.bfloat16, dict(T=1.0)),
    ("conf_random_len", 24, 8, 4, 4099, torch.bfloat16, dict(T=1.0, draft_len="random")),
    ("winner", 16, 4, 3, 3001, torch.bfloat16, dict(T=1.0, wm=cv.W_WINNER)),
    ("point", 16, 4, 2, 3001, torch.bfloat16, dict(T=1.0, wm=cv.W_POINT)),
    ("greedy", 16, 4, 3, 3001, torch.bfloat16, dict(T=0.0)),
    ("temp07_f32", 12, 4, 2, 2053, torch.float32, dict(T=0.7)),
    ("logits", 12, 4, 3, 2053, torch.float32, dict(T=1.0, draft_kind="logits")),
    ("unaligned_split", 16, 5, 3, 5003, torch.bfloat16, dict(T=1.0, split="odd")),
    ("errors", 16, 4, 3, 3001, torch.bfloat16, dict(T=1.0, inject=True)),
]
# BASELINE config c5 at full size (B = 1024, V = 128256): run with --c5
C5_CASE = ("c5_full", 1024, 8, 4, 128256, torch.bfloat16, dict(T=1.0, gpu_gen=True))


def make_inputs(B, k, N, V, dtype, kw, seed):
    if kw.get("gpu_gen"):  # large cases: generated on the GPU in request slices of 64
        dev = torch.device("cuda", torch.cuda.current_device())
        parts = [synth.linear_inputs(64, k, N, V, dtype=dtype, seed=seed + b0, device=dev, rid_base=b0)
                 for b0 in range(0, B, 64)]
        return dict(target=torch.cat([p["target"] for p in parts]), draft=torch.cat([p["draft"] for p in parts]),
                    draft_tokens=torch.cat([p["draft_tokens"] for p in parts]),
                    request_ids=torch.cat([p["request_ids"] for p in parts]), draft_len=None, V=V,
                    ld=parts[0]["ld"])
    dl = "random" if kw.get("draft_len") == "random" else None
    inp = synth.linear_inputs(B, k, N, V, dtype=dtype, seed=seed, draft_len=dl,
                              draft_kind=kw.get("draft_kind", "probs"))
    if kw.get("inject"):
        inp["draft_tokens"][1, 0, 0] = V + 3           # token out of range (global check)
        inp["target"][3, 1, V - 2] = float("nan")       # non-finite in the last shard
        inp["draft"][5, 0, 1, 7] = float("nan")         # non-finite in the first shard
    return inp


def run_case(name, B, k, N, V, dtype, kw, world, rank, dev):
    seed = 1000 + sum(map(ord, name))
    inp = make_inputs(B, k, N, V, dtype, kw, seed)
    if kw.get("split") == "odd":
        edges = [0] + [V * r // world + (5 if r % 2 else 3) for r in range(1, world)] + [V]  # not 8-aligned
        b, e = edges[rank], edges[rank + 1]
    else:
        b, e = vocab_shard(V, world, rank)
    T = kw.get("T", 1.0)
    wm = kw.get("wm", cv.W_CONF)
    dk = cv.DRAFT_LOGITS if kw.get("draft_kind") == "logits" else cv.DRAFT_PROBS
    obj = [cv.cosine_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = cv.cosine_verify_init(V, device=dev.index, max_batch=B, max_draft_len=k, max_drafters=N,
                                target_dtype=dtype, draft_dtype=dtype, draft_kind=dk, seed=7,
                                nranks=world, rank=rank, vocab_begin=b, vocab_end=e,
                                nccl_unique_id=obj[0])
    ver = cv.Verifier(V, max_batch=B, k=k, N=N, device=dev.index, debug=True, ctx=ctx)
    tgt = column_shard(inp["target"][..., :V], b, e).to(dev)
    drf = column_shard(inp["draft"][..., :V], b, e).to(dev)
    dl = inp["draft_len"].to(dev) if inp["draft_len"] is not None else None
    a, o, s = ver.verify(tgt, drf, inp["draft_tokens"].to(dev), inp["request_ids"].to(dev),
                         temperature=T, draft_len=dl, weight_mode=wm)
    torch.cuda.synchronize(dev)
    g = dict(accept_len=a.cpu().numpy().copy(), out_tokens=o.cpu().numpy().copy(),
             status=s.cpu().numpy().copy(), launches=cv.cosine_last_launch_count(ver.ctx))
    for n, t in ver.debug.items():
        g[n] = t[:B].cpu().numpy().copy()
    exchange = cv.cosine_exchange_mode(ctx)
    ver.close()
    # every rank must hold the same outputs
    mine = torch.tensor(np.concatenate([g["accept_len"], g["out_tokens"].ravel(), g["status"]]), dtype=torch.int64)
    allv = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine)
    replicated = all(bool((x == allv[0]).all()) for x in allv)
    res = dict(case=name, shard=[b, e], replicated=replicated, launches=g["launches"],
               exchange=exchange)
    if rank != 0:
        return res
    import parity
    r = parity.oracle_verify(inp, T=T, seed=7, wm=wm, draft_kind=kw.get("draft_kind", "probs"))
    nm, nf = parity.compare(g, r, greedy=(T == 0.0), check_probs=not kw.get("inject"))
    u = parity.gpu_verify(inp, T=T, seed=7, wm=wm, draft_kind=kw.get("draft_kind", "probs"), device=dev.index)
    diff = np.nonzero((u["accept_len"] != g["accept_len"]) | (u["out_tokens"] != g["out_tokens"]).any(1)
                      | ((u["status"] & 0xff) != (g["status"] & 0xff)))[0]
    flagged = (r["tie_margin"] < parity.TIE) | ((g["status"] & 0x200) != 0) | ((u["status"] & 0x200) != 0)
    unflagged = [int(i) for i in diff if not flagged[i]]
    assert not unflagged, f"{name}: sharded != unsharded at {unflagged[:5]}"
    assert replicated, f"{name}: outputs differ across ranks"
    res.update(oracle_mismatch=nm, oracle_flagged=nf, unsharded_diff=len(diff),
               mean_accept=float(np.mean(g["accept_len"][g["accept_len"] >= 0])) if (g["accept_len"] >= 0).any() else None)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--c5", action="store_true", help="also run BASELINE config c5 at full size")
    args = ap.parse_args()
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    results, ok = [], True
    for name, B, k, N, V, dtype, kw in CASES + ([C5_CASE] if args.c5 else []):
        try:
            results.append(run_case(name, B, k, N, V, dtype, kw, world, rank, dev))
        except Exception as ex:  # keep the ranks in step: report and go on
            ok = False
            results.append(dict(case=name, error=f"{type(ex).__name__}: {ex}",
                                trace=traceback.format_exc()[-2000:]))
    flags = torch.tensor([int(ok)])
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    ok = bool(flags.item())
    if rank == 0:
        summary = dict(world=world, ok=ok, results=results)
        txt = json.dumps(summary, indent=1, default=str)
        print(txt)
        if args.out:
            with open(args.out, "w") as f:
                f.write(txt)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
