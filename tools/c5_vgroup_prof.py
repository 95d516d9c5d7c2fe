"""c5 at G ranks as a one-GPU virtual group (same sharded kernels, device copies for the
exchanges): run a few calls so that `ncu` can list every kernel's duration per rank."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_10325_b200 as cv  # noqa: E402
import synth  # noqa: E402
from paper_2503_10325_b200.sharding import vocab_shard  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = synth.CONFIGS["c5"]
B, N, k, V = c["B"], c["N"], c["k"], c["V"]
dev = torch.device("cuda", 0)
shards = [vocab_shard(V, G, r) for r in range(G)]
width = max(e - b for b, e in shards)
ld = (width + 7) // 8 * 8
tg, dr = [], []
for r, (b0, e0) in enumerate(shards):
    inp = synth.linear_inputs(B, k, N, e0 - b0, dtype=c["dtype"], seed=77 + r, device=dev)
    t = torch.zeros((B, k + 1, ld), dtype=c["dtype"], device=dev)
    d = torch.zeros((B, k, N, ld), dtype=c["dtype"], device=dev)
    t[..., :e0 - b0] = inp["target"][..., :e0 - b0]
    d[..., :e0 - b0] = inp["draft"][..., :e0 - b0]
    tg.append(t)
    dr.append(d)
    toks = (inp["draft_tokens"] + b0).clamp_(max=V - 1)
    rids = inp["request_ids"]
    del inp
ctxs = cv.cosine_verify_init_vgroup(V, shards, max_batch=B, max_draft_len=k, max_drafters=N, target_dtype=c["dtype"],
                                    draft_dtype=c["dtype"], seed=1)
al = [torch.empty(B, dtype=torch.int32, device=dev) for _ in range(G)]
ot = [torch.empty(B, k + 1, dtype=torch.int32, device=dev) for _ in range(G)]
st = [torch.empty(B, dtype=torch.int32, device=dev) for _ in range(G)]
for _ in range(3):
    cv.cosine_verify_batch_vgroup(ctxs, tg, dr, toks, rids, al, ot, st, temperature=1.0,
                                  peer_exchange="peer" in sys.argv)
torch.cuda.synchronize()
print("ok", G, cv.cosine_last_launch_count(ctxs[0]))
