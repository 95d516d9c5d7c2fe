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


def tree_shape(schedule=(4, 2, 2, 1, 1, 1, 1, 1), cap: int = 64):
    """Breadth-first draft tree: every node at depth d gets schedule[d] children until `cap`
    non-root nodes exist (c4: level sizes 1/4/8/16/16/16/4, 49 internal nodes).  Returns
    (parent list, internal-row list) with children in ascending node id."""
    parent = [-1]
    depth = [0]
    frontier = [0]
    while frontier and len(parent) - 1 < cap:
        nxt = []
        for node in frontier:
            d = depth[node]
            if d >= len(schedule):
                continue
            for _ in range(schedule[d]):
                if len(parent) - 1 >= cap:
                    break
                parent.append(node)
                depth.append(d + 1)
                nxt.append(len(parent) - 1)
        frontier = nxt
    has_child = [False] * len(parent)
    for c in range(1, len(parent)):
        has_child[parent[c]] = True
    irow, n_int = [], 0
    for j in range(len(parent)):
        if has_child[j]:
            irow.append(n_int)
            n_int += 1
        else:
            irow.append(-1)
    return parent, irow


def tree_inputs(B: int, N: int, V: int, *, schedule=(4, 2, 2, 1, 1, 1, 1, 1), cap: int = 64,
                dtype=torch.bfloat16, seed: int = 0, device="cpu", sigma: float = 5.0,
                rho_hi: float = 0.99, rho_lo: float = 0.95, ld: int | None = None, rid_base: int = 0,
                chunk: int = 8, pad_value: float = float("nan")):
    """Tree-shaped drafts (config c4).  Every node j has its own target row (the target after the
    path to j) and every internal node N drafter rows (same recipe as linear_inputs); the drafters'
    own tokens X_n ~ their rows; a node's children are drawn WITHOUT replacement from the plain
    average of its drafter rows (input synthesis: this is not the method's fused q)."""
    parent, irow = tree_shape(schedule, cap)
    nn = len(parent)
    I = sum(1 for r in irow if r >= 0)
    align = 16 // torch.tensor([], dtype=dtype).element_size()
    ld = ld or _round_up(V, align)
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    target = torch.full((B, nn, ld), pad_value, dtype=dtype, device=dev)
    draft = torch.full((B, max(I, 1), N, ld), pad_value, dtype=dtype, device=dev)
    ndt = torch.zeros((B, max(I, 1), N), dtype=torch.int32, device=dev)
    tok = torch.zeros((B, nn), dtype=torch.int32, device=dev)
    rids = torch.arange(rid_base, rid_base + B, dtype=torch.int64, device=dev)
    inodes = [j for j in range(nn) if irow[j] >= 0]
    kids = {j: [c for c in range(1, nn) if parent[c] == j] for j in inodes}
    for b0 in range(0, B, chunk):
        b1 = min(B, b0 + chunk)
        nb = b1 - b0
        z = torch.randn((nb, nn, V), generator=gen, device=dev, dtype=torch.float32)
        target[b0:b1, :, :V] = (sigma * z).to(dtype)
        if I:
            eps = torch.randn((nb, I, N, V), generator=gen, device=dev, dtype=torch.float32)
            dom = (rids[b0:b1] % N).view(nb, 1, 1, 1)
            n_idx = torch.arange(N, device=dev).view(1, 1, N, 1)
            rho = torch.where(n_idx == dom, torch.tensor(rho_hi, device=dev), torch.tensor(rho_lo, device=dev))
            noise = torch.sqrt(torch.clamp(1.0 - rho * rho, min=0.0))
            zi = z[:, inodes, None, :]
            rows = torch.softmax(sigma * (rho * zi + noise * eps), dim=-1).to(dtype)
            del eps, zi
            draft[b0:b1, :I, :, :V] = rows
            flat = rows.reshape(-1, V).float()
            ndt[b0:b1, :I] = torch.multinomial(flat, 1, generator=gen).view(nb, I, N).to(torch.int32)
            avg = rows.float().mean(dim=2)  # [nb][I][V]
            for r, j in enumerate(inodes):
                m = len(kids[j])
                ch = torch.multinomial(avg[:, r], m, replacement=False, generator=gen)
                for s_i, c in enumerate(kids[j]):
                    tok[b0:b1, c] = ch[:, s_i].to(torch.int32)
            del rows, flat, avg
        del z
    par_t = torch.tensor(parent, dtype=torch.int32, device=dev).expand(B, nn).contiguous()
    irow_t = torch.tensor(irow, dtype=torch.int32, device=dev).expand(B, nn).contiguous()
    return dict(parent=par_t, node_token=tok, internal_row=irow_t, target=target, draft=draft,
                node_draft_tokens=ndt, request_ids=rids, V=V, ld=ld, J=nn - 1, I=I)


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


def tree_algorithmic_bytes(B: int, nn: int, I: int, N: int, V: int, t_bytes: int, q_bytes: int) -> int:
    """All-nodes accounting: every node's target row and every internal node's
    drafter rows read once, plus the tree arrays and the outputs."""
    return B * (nn * V * t_bytes + I * N * V * q_bytes + 4 * nn * 3 + 4 * I * N + 8 + 4 * (2 * nn + 2))


__all__ = ["CONFIGS", "linear_inputs", "tiny_inputs", "tree_shape", "tree_inputs", "algorithmic_bytes",
           "tree_algorithmic_bytes", "verified_tokens", "describe"]
