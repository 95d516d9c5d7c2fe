"""Seeded synthetic inputs shaped like the paper's Llama-family workloads.

This module is shared by the tests, bench.py and the oracle checks, and it holds
NONE of the verification method's arithmetic: it only draws random logits,
turns the drafters' logits into the probability rows a drafter would ship
(input synthesis, not the method), and samples the drafters' own tokens with
torch's RNG (not Philox, not the inverse CDF of the method).

Recipe:
* target logits  l = sigma * z, z ~ N(0, 1), sigma = 5 (median top-1 prob ~0.3);
* drafter n at request b: l_n = sigma * (rho z + sqrt(1 - rho^2) eps_n) (variance
  preserving, so noisier drafters are flatter and lose the confidence argmax, as in
  Fig. 3b), rho = rho_hi if n == domain(b) = rid mod N else rho_lo (domain
  specialised drafters, Table 2's diagonal P:701-705, Fig. 3a);
* drafter rows: PROBS = dtype(softmax(l_n)) or LOGITS = dtype(l_n);
* drafter tokens X_n ~ its own (rounded) row (or its argmax: greedy drafting);
* row padding columns [V, ld) are NaN so any read past the vocabulary is caught.
"""
from __future__ import annotations

import math

import torch

CONFIGS = {
    # name: (B, N, k, V, dtype) — BASELINE.json configs[0..4]
    "c1": dict(B=1, N=2, k=4, V=32000, dtype=torch.float32),
    "c2": dict(B=64, N=3, k=8, V=32000, dtype=torch.bfloat16),
    "c3": dict(B=256, N=4, k=8, V=128256, dtype=torch.bfloat16),
    "c4": dict(B=128, N=4, k=8, V=128256, dtype=torch.bfloat16, tree_nodes=64),
    "c5": dict(B=1024, N=4, k=8, V=128256, dtype=torch.bfloat16, shards=8),
}


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def linear_inputs(B: int, k: int, N: int, V: int, *, dtype=torch.bfloat16, draft_dtype=None,
                  seed: int = 0, device="cpu", sigma: float = 5.0, rho_hi: float = 0.99,
                  rho_lo: float = 0.95, ld: int | None = None, draft_len=None, rid_base: int = 0,
                  draft_kind: str = "probs", token_mode: str = "sample", chunk: int = 32,
                  pad_value: float = float("nan")):
    """Returns dict(target [B][k+1][ld], draft [B][k][N][ld], draft_tokens [B][k][N] int32,
    request_ids [B] int64 (global ids rid_base + b), draft_len [B] int32 or None)."""
    draft_dtype = draft_dtype or dtype
    align = 16 // min(torch.tensor([], dtype=dtype).element_size(),
                      torch.tensor([], dtype=draft_dtype).element_size())
    ld = ld or _round_up(V, align)
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    target = torch.full((B, k + 1, ld), pad_value, dtype=dtype, device=dev)
    draft = torch.full((B, k, N, ld), pad_value, dtype=draft_dtype, device=dev)
    tokens = torch.empty((B, k, N), dtype=torch.int32, device=dev)
    rids = torch.arange(rid_base, rid_base + B, dtype=torch.int64, device=dev)
    for b0 in range(0, B, chunk):
        b1 = min(B, b0 + chunk)
        nb = b1 - b0
        z = torch.randn((nb, k + 1, V), generator=gen, device=dev, dtype=torch.float32)
        target[b0:b1, :, :V] = (sigma * z).to(dtype)
        eps = torch.randn((nb, k, N, V), generator=gen, device=dev, dtype=torch.float32)
        dom = (rids[b0:b1] % N).view(nb, 1, 1, 1)
        n_idx = torch.arange(N, device=dev).view(1, 1, N, 1)
        rho = torch.where(n_idx == dom, torch.tensor(rho_hi, device=dev), torch.tensor(rho_lo, device=dev))
        noise = torch.sqrt(torch.clamp(1.0 - rho * rho, min=0.0))
        dl = sigma * (rho * z[:, :k, None, :] + noise * eps)
        del eps
        if draft_kind == "probs":
            rows = torch.softmax(dl, dim=-1).to(draft_dtype)
        else:
            rows = dl.to(draft_dtype)
        draft[b0:b1, :, :, :V] = rows
        flat = rows.reshape(-1, V).float()
        if draft_kind != "probs":
            flat = torch.softmax(flat, dim=-1)
        if token_mode == "argmax":
            tok = torch.argmax(flat, dim=-1)
        else:
            tok = torch.multinomial(flat, 1, generator=gen).squeeze(-1)
        tokens[b0:b1] = tok.view(nb, k, N).to(torch.int32)
        del dl, rows, flat, z
    dlen = None
    if draft_len is not None:
        if isinstance(draft_len, str) and draft_len == "random":
            dlen = torch.randint(1, k + 1, (B,), generator=gen, device=dev, dtype=torch.int64).to(torch.int32)
        else:
            dlen = torch.as_tensor(draft_len, dtype=torch.int32, device=dev).expand(B).clone()
    return dict(target=target, draft=draft, draft_tokens=tokens, request_ids=rids, draft_len=dlen,
                V=V, ld=ld)


def tiny_inputs(B: int, k: int, N: int, V: int, *, seed: int = 0, sigma: float = 1.0, ld=None,
                dtype=torch.float32, rho=0.5):
    """Small-vocabulary inputs (V = 2..16) for distribution tests: the same recipe, flatter."""
    return linear_inputs(B, k, N, V, dtype=dtype, seed=seed, sigma=sigma, rho_hi=rho, rho_lo=rho,
                         ld=ld, chunk=max(B, 1))


def algorithmic_bytes(B: int, k: int, N: int, V: int, t_bytes: int, q_bytes: int,
                      draft_len=None) -> int:
    """Every input byte read once + the outputs: rows 0..gamma_b of the target
    and the drafter rows of positions < gamma_b, tokens, ids, outputs."""
    if draft_len is None:
        g_sum = B * k
    else:
        g_sum = int(torch.as_tensor(draft_len).sum())
    rows_t = g_sum + B
    rows_q = g_sum * N
    return rows_t * V * t_bytes + rows_q * V * q_bytes + 4 * g_sum * N + 8 * B + 4 * B * (k + 2) + 4 * B


def verified_tokens(B: int, k: int, draft_len=None) -> int:
    return B * k if draft_len is None else int(torch.as_tensor(draft_len).sum())


def describe(name: str) -> dict:
    c = dict(CONFIGS[name])
    c["dtype"] = str(c["dtype"]).replace("torch.", "")
    return c


__all__ = ["CONFIGS", "linear_inputs", "tiny_inputs", "algorithmic_bytes", "verified_tokens",
           "describe"]
