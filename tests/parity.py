"""Helpers shared by the GPU parity tests: run the CUDA path and the oracle on the same
seeded inputs and compare (test infrastructure; imports the oracle)."""
from __future__ import annotations

import json
import os

import numpy as np
import torch

import oracle

TIE = 1e-6        # north_star: ties within 1e-6 of a threshold are flagged, not failures
PROB_RTOL = 1e-5  # north_star: probabilities within 1e-5 relative (fp32)
MAX_FLAG_FRAC = 0.01  # a flagged near tie is rare (margins < 1e-6); more than 1% means a regression
# SAMPLE selection draws x*_i ~ q_i at every position (k draws per request, not one): a draw that
# lands in a bin of mass < 1e-6 (absolute, ~V^-1 for V = 128256) is flagged, so ~k times more
# requests are flagged (measured: 8 of 256 at c3); the bound scales with the draws
MAX_FLAG_FRAC_SAMPLE = 0.05


def record(name, **counts):
    """Append one line of parity counts to $PARITY_LOG (GPU runs collect them for DESIGN.md)."""
    path = os.environ.get("PARITY_LOG")
    line = dict(test=os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], case=name, **counts)
    print("parity:", json.dumps(line))
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(line) + "\n")


def gpu_verify(inp, *, T=1.0, seed=7, step=0, wm=0, sm=0, draft_kind="probs", cluster_size=0,
               device=0, subset=None, lazy=False):
    import paper_2503_10325_b200 as cv
    tgt, drf = inp["target"], inp["draft"]
    B, kp1, _ = tgt.shape
    N = drf.shape[2]
    dev = torch.device("cuda", device)
    ver = cv.Verifier(inp["V"], max_batch=B, k=kp1 - 1, N=N, device=device, target_dtype=tgt.dtype,
                      draft_dtype=drf.dtype, seed=seed, debug=True, cluster_size=cluster_size,
                      draft_kind=cv.DRAFT_LOGITS if draft_kind == "logits" else cv.DRAFT_PROBS)
    d = {n: (t.to(dev) if torch.is_tensor(t) else t) for n, t in inp.items()}
    a, o, s = ver.verify(d["target"], d["draft"], d["draft_tokens"], d["request_ids"], temperature=T,
                         draft_len=d["draft_len"], step=step, weight_mode=wm, select_mode=sm, lazy=lazy)
    torch.cuda.synchronize()
    out = dict(accept_len=a.cpu().numpy().copy(), out_tokens=o.cpu().numpy().copy(),
               status=s.cpu().numpy().copy(), launches=cv.cosine_last_launch_count(ver.ctx))
    for n, t in ver.debug.items():
        out[n] = t[:B].cpu().numpy().copy()
    ver.close()
    return out


def oracle_verify(inp, *, T=1.0, seed=7, step=0, wm=0, sm=0, draft_kind="probs", subset=None):
    sel = slice(None) if subset is None else subset
    dl = inp["draft_len"]
    return oracle.verify_batch_parallel(inp["target"][sel].cpu(), inp["draft"][sel].cpu(),
                               inp["draft_tokens"][sel].cpu(), inp["request_ids"][sel].cpu(),
                               temperature=T, seed=seed, step=step,
                               draft_len=None if dl is None else dl[sel].cpu(),
                               draft_kind=oracle.DRAFT_LOGITS if draft_kind == "logits" else oracle.DRAFT_PROBS,
                               weight_mode=wm, select_mode=sm, vocab=inp["V"])


def compare(g, r, subset=None, check_probs=True, greedy=False, name="", max_flag_frac=MAX_FLAG_FRAC):
    """Bit-exact accept_len / out_tokens / status except where the oracle flags a near tie; the
    flagged requests are counted and bounded (MAX_FLAG_FRAC)."""
    idx = np.arange(len(r["accept_len"])) if subset is None else np.asarray(subset)
    ga, go, gs = g["accept_len"][idx], g["out_tokens"][idx], g["status"][idx]
    assert (gs & 0xff == r["status"] & 0xff).all(), (gs, r["status"])
    mism = np.nonzero((ga != r["accept_len"]) | (go != r["out_tokens"]).any(1))[0]
    flagged = r["tie_margin"] < TIE
    bad = [int(b) for b in mism if not flagged[b]]
    nflag = int(flagged.sum())
    record(name, requests=int(len(idx)), mismatches=int(len(mism)), unflagged_mismatches=len(bad),
           flagged=nflag)
    assert nflag <= max(1, max_flag_frac * len(idx)), f"{nflag} of {len(idx)} requests flagged as near ties"
    assert not bad, f"unflagged mismatches at {bad[:5]}: gpu {ga[bad[0]]} {go[bad[0]]} " \
                    f"oracle {r['accept_len'][bad[0]]} {r['out_tokens'][bad[0]]} margin {r['tie_margin'][bad[0]]}"
    if check_probs:
        ok = (r["status"] & 0xff) == 0
        pairs = [("q_x", "q_x"), ("draft_norm", "sigma"), ("conf", "conf"), ("weights", "weights")]
        if not greedy:  # T = 0 has no softmax statistics
            pairs += [("p_x", "p_x"), ("row_sumexp", "S")]
        # p(x*), q(x*) are values AT the fused token: compare them where both sides fused the same
        # token.  Under SAMPLE selection a position after the first rejection is not on the
        # realised path (its draw is discarded), so a near tie there may pick another token
        # without being flagged; on the path (positions < L) the tokens are equal (checked above).
        same_x = g["fused_tokens"][idx][ok] == r["fused_tokens"][ok]
        L = r["accept_len"][ok]
        on_path = (np.arange(same_x.shape[1])[None, :] < L[:, None]) & ~flagged[ok][:, None]
        assert same_x[on_path].all()
        for gk, rk in pairs:
            gv, rv = g[gk][idx][ok], r[rk][ok]
            m = np.isfinite(rv) & (np.abs(rv) > 1e-30)
            if rk in ("q_x", "p_x"):
                m &= same_x
            if rk == "S":
                m &= rv > 0
            if m.any():
                rel = np.abs(gv[m] - rv[m]) / np.abs(rv[m])
                assert rel.max() < PROB_RTOL, f"{gk}: max rel err {rel.max():.3g}"
    return len(mism), int(flagged.sum())
