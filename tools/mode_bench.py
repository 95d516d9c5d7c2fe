"""c3-shaped timing of the verify modes that bench.py does not expose (LOGITS drafts, SAMPLE
selection): CUDA events around each call, inputs > L2.  Prints one JSON line per mode."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10325_b200 as cv  # noqa: E402
import synth  # noqa: E402

c = synth.CONFIGS["c3"]
B, N, k, V = c["B"], c["N"], c["k"], c["V"]
dev = torch.device("cuda", 0)
for kind, sm in (("logits", cv.SEL_ARGMAX), ("logits", cv.SEL_SAMPLE), ("probs", cv.SEL_SAMPLE)):
    inp = synth.linear_inputs(B, k, N, V, dtype=c["dtype"], seed=5, device=dev, draft_kind=kind)
    ver = cv.Verifier(V, max_batch=B, k=k, N=N, seed=1,
                      draft_kind=cv.DRAFT_LOGITS if kind == "logits" else cv.DRAFT_PROBS)
    f = lambda: ver.verify(inp["target"], inp["draft"], inp["draft_tokens"], inp["request_ids"], select_mode=sm)
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(json.dumps({"drafts": kind, "select": "sample" if sm else "argmax", "us_per_call": round(us, 1),
                      "verified_tokens_per_s": B * k / (us / 1e6)}))
    ver.close()
    del inp
    torch.cuda.empty_cache()
