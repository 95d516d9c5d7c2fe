"""Vocabulary-sharded verification on ONE GPU: G contexts of a virtual
group (cosine_verify_init_vgroup) run the sharded kernels and record layouts of the NCCL path, with every all-gather replaced by device copies in rank order
(cosine_verify_batch_vgroup).  Every rank's outputs must be identical, equal to the unsharded call
on the full rows (up to flagged near ties: the row sums are re-associated) and to the oracle.
The same cases run over NCCL on 2 / 4 GPUs in test_gpu_vocab_shard.py."""
import os
import sys

import numpy as np
import pytest
import torch

import synth
from paper_2503_10325_b200.sharding import vocab_shard

from . import parity

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import shard_check  # noqa: E402  (the case list and the column-shard helper)

pytestmark = pytest.mark.gpu


def _vgroup_verify(inp, shards, *, T=1.0, wm=0, draft_kind="probs", seed=7, dev=None, peer=False):
    """Run the virtual group over the column shards of `inp`; returns one output dict per rank."""
    import paper_2503_10325_b200 as cv
    dev = dev or torch.device("cuda", 0)
    B, kp1, _ = inp["target"].shape
    k, N, V = kp1 - 1, inp["draft"].shape[2], inp["V"]
    dt, qt = inp["target"].dtype, inp["draft"].dtype
    dk = cv.DRAFT_LOGITS if draft_kind == "logits" else cv.DRAFT_PROBS
    ctxs = cv.cosine_verify_init_vgroup(V, shards, max_batch=B, max_draft_len=k, max_drafters=N, target_dtype=dt,
                                        draft_dtype=qt, draft_kind=dk, seed=seed)
    reps = 2 if peer else 1  # (peer: a second call checks that the arrival targets advance)
    width = max(e - b for b, e in shards)
    ld = (width + 7) // 8 * 8
    tg, dr = [], []
    for b, e in shards:
        t = torch.full((B, kp1, ld), float("nan"), dtype=dt, device=dev)
        d = torch.full((B, k, N, ld), float("nan"), dtype=qt, device=dev)
        t[..., :e - b] = inp["target"][..., b:e].to(dev)
        d[..., :e - b] = inp["draft"][..., b:e].to(dev)
        tg.append(t)
        dr.append(d)
    G = len(shards)
    al = [torch.empty(B, dtype=torch.int32, device=dev) for _ in range(G)]
    ot = [torch.empty(B, kp1, dtype=torch.int32, device=dev) for _ in range(G)]
    st = [torch.empty(B, dtype=torch.int32, device=dev) for _ in range(G)]
    dl = inp["draft_len"].to(dev) if inp["draft_len"] is not None else None
    for _ in range(reps):
        cv.cosine_verify_batch_vgroup(ctxs, tg, dr, inp["draft_tokens"].to(dev), inp["request_ids"].to(dev), al, ot,
                                      st, temperature=T, draft_len=dl, weight_mode=wm, peer_exchange=peer)
    torch.cuda.synchronize()
    launches = cv.cosine_last_launch_count(ctxs[0])
    for c in ctxs:
        cv.cosine_verify_destroy(c)
    return [dict(accept_len=a.cpu().numpy(), out_tokens=o.cpu().numpy(), status=s.cpu().numpy(), launches=launches)
            for a, o, s in zip(al, ot, st)]


def _check(name, inp, outs, *, T=1.0, wm=0, draft_kind="probs", oracle_slices=None):
    for g in outs[1:]:  # replicated on every rank
        for n in ("accept_len", "out_tokens", "status"):
            np.testing.assert_array_equal(g[n], outs[0][n])
    g = outs[0]
    u = parity.gpu_verify(inp, T=T, seed=7, wm=wm, draft_kind=draft_kind)
    r = parity.oracle_verify(inp, T=T, seed=7, wm=wm, draft_kind=draft_kind)
    parity.compare(g, r, greedy=(T == 0.0), check_probs=False, name=name)
    diff = (u["accept_len"] != g["accept_len"]) | (u["out_tokens"] != g["out_tokens"]).any(1) | \
        ((u["status"] & 0xff) != (g["status"] & 0xff))
    flagged = (r["tie_margin"] < parity.TIE) | ((g["status"] & 0x200) != 0) | ((u["status"] & 0x200) != 0)
    assert not (diff & ~flagged).any(), f"{name}: sharded != unsharded at {np.nonzero(diff & ~flagged)[0][:5]}"


@pytest.mark.parametrize("peer", [False, True], ids=["copies", "peer"])
@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("case", shard_check.CASES, ids=[c[0] for c in shard_check.CASES])
def test_vgroup_cases(cuda_ok, case, G, peer):
    name, B, k, N, V, dtype, kw = case
    inp = shard_check.make_inputs(B, k, N, V, dtype, kw, 1000 + sum(map(ord, name)))
    if kw.get("split") == "odd":
        edges = [0] + [V * r // G + (5 if r % 2 else 3) for r in range(1, G)] + [V]  # not 8-aligned
        shards = [(edges[r], edges[r + 1]) for r in range(G)]
    else:
        shards = [vocab_shard(V, G, r) for r in range(G)]
    T, wm, dk = kw.get("T", 1.0), kw.get("wm", 0), kw.get("draft_kind", "probs")
    outs = _vgroup_verify(inp, shards, T=T, wm=wm, draft_kind=dk, peer=peer)
    _check(f"vgroup {name} G={G}{' peer' if peer else ''}", inp, outs, T=T, wm=wm, draft_kind=dk)


@pytest.mark.parametrize("peer", [False, True], ids=["copies", "peer"])
def test_vgroup_c5_full_size(cuda_ok, peer):
    # BASELINE config c5: B = 1024, k = 8, N = 4, V = 128256 split over G = 8 shards of 16032
    # columns — the sharded kernels at their real shape (9216 units per record exchange), every
    # request checked against the oracle and the unsharded call.
    c = synth.CONFIGS["c5"]
    B, N, k, V, G = c["B"], c["N"], c["k"], c["V"], c["shards"]
    dev = torch.device("cuda", 0)
    parts = [synth.linear_inputs(64, k, N, V, dtype=c["dtype"], seed=5000 + b0, device=dev, rid_base=b0)
             for b0 in range(0, B, 64)]
    inp = dict(target=torch.cat([p["target"] for p in parts]), draft=torch.cat([p["draft"] for p in parts]),
               draft_tokens=torch.cat([p["draft_tokens"] for p in parts]),
               request_ids=torch.cat([p["request_ids"] for p in parts]), draft_len=None, V=V, ld=parts[0]["ld"])
    del parts
    shards = [vocab_shard(V, G, r) for r in range(G)]
    assert all(e - b == 16032 for b, e in shards)
    outs = _vgroup_verify(inp, shards, peer=peer)
    assert outs[0]["launches"] == 6
    _check(f"vgroup c5 G=8{' peer' if peer else ''}", inp, outs)
