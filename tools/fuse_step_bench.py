"""Timing of cosine_fuse_step (NEXT-2) on B200: B requests x N drafter LM-head rows per call,
CUDA events on the launching stream, inputs larger than L2 (no flush needed).  Prints one JSON
line (not the bench.py contract line; the drafter-side step is not the north_star metric)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10325_b200 as cv  # noqa: E402


def main(B=256, N=4, V=128256, steps=50, warmup=5):
    dev = torch.device("cuda", 0)
    x = (5.0 * torch.randn(B, N, V, device=dev)).to(torch.bfloat16)
    ctx = cv.cosine_verify_init(V, max_batch=B, max_draft_len=N, max_drafters=N, draft_dtype=torch.bfloat16)
    own = torch.empty(B, N, dtype=torch.int32, device=dev)
    conf = torch.empty(B, N, dtype=torch.float32, device=dev)
    fused = torch.empty(B, dtype=torch.int32, device=dev)
    win = torch.empty(B, dtype=torch.int32, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    for _ in range(warmup):
        cv.cosine_fuse_step(ctx, x, own, conf, fused, win, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        cv.cosine_fuse_step(ctx, x, own, conf, fused, win, st)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / steps * 1e3
    nbytes = B * N * V * 2
    print(json.dumps({"op": "cosine_fuse_step", "B": B, "N": N, "V": V, "dtype": "bf16", "us_per_call": us,
                      "fused_positions_per_s": B / (us / 1e6), "bytes_per_call": nbytes,
                      "achieved_GBps": nbytes / (us / 1e6) / 1e9, "peak_GBps": 6550.4,
                      "frac": nbytes / (us / 1e6) / 1e9 / 6550.4}))
    cv.cosine_verify_destroy(ctx)


if __name__ == "__main__":
    main()
