"""GPU parity of the two other C-ABI entry points: cosine_fuse_drafts (Eq. 4 fusion alone)
and cosine_sample_residual (the final-token sample)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("wm,sm", [(0, 0), (1, 0), (2, 0), (3, 0), (0, 1)])
def test_fuse_drafts(cuda_ok, wm, sm):
    import paper_2503_10325_b200 as cv
    B, k, N, V = 12, 5, 3, 3001
    inp = synth.linear_inputs(B, k, N, V, dtype=torch.bfloat16, seed=200 + wm)
    dev = torch.device("cuda", 0)
    ctx = cv.cosine_verify_init(V, max_batch=B, max_draft_len=k, max_drafters=N, seed=3)
    ld = inp["ld"]
    ft = torch.empty(B, k, dtype=torch.int32, device=dev)
    w = torch.empty(B, k, N, device=dev)
    sg = torch.empty(B, k, N, device=dev)
    fq = torch.empty(B, k, ((V + 3) // 4) * 4, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    cv.cosine_fuse_drafts(ctx, inp["draft"].to(dev), inp["draft_tokens"].to(dev), inp["request_ids"].to(dev),
                          ft, st, weight_mode=wm, select_mode=sm, weights=w, draft_norm=sg, fused_q=fq, step=2)
    torch.cuda.synchronize()
    r = oracle.fuse_drafts(inp["draft"], inp["draft_tokens"], inp["request_ids"], seed=3, step=2,
                           weight_mode=wm, select_mode=sm, want_q=True, vocab=V)
    cv.cosine_verify_destroy(ctx)
    flagged = r["tie_margin"] < 1e-6
    bad = (ft.cpu().numpy() != r["fused_tokens"]).any(1) & ~flagged
    assert not bad.any()
    np.testing.assert_array_equal(st.cpu().numpy() & 0xff, r["status"])
    np.testing.assert_allclose(w.cpu().numpy(), r["weights"], rtol=1e-5)
    np.testing.assert_allclose(sg.cpu().numpy(), r["draft_norm"], rtol=1e-5)
    np.testing.assert_allclose(fq.cpu().numpy()[..., :V], r["fused_q"], rtol=1e-5, atol=1e-9)


@pytest.mark.parametrize("with_stats,with_draft,T", [(False, True, 1.0), (True, True, 1.0), (False, False, 1.0),
                                                     (True, True, 0.7), (True, False, 0.7), (False, True, 0.7)])
def test_sample_residual(cuda_ok, with_stats, with_draft, T):
    import paper_2503_10325_b200 as cv
    B, N, V = 64, 3, 5003
    inp = synth.linear_inputs(B, 1, N, V, dtype=torch.bfloat16, seed=300)
    dev = torch.device("cuda", 0)
    rows = inp["target"][:, 0].contiguous()
    drafts = inp["draft"][:, 0].contiguous()
    rng = np.random.default_rng(0)
    wts = torch.tensor(rng.dirichlet(np.ones(N), size=B), dtype=torch.float32)
    norms = drafts[..., :V].float().sum(-1)
    nodes = torch.tensor(rng.integers(0, 8, B), dtype=torch.int32)
    rm = rs = None
    if with_stats:
        l = rows[:, :V].double()
        rm = l.max(-1).values.float()
        rs = torch.exp((l - rm.double()[:, None]) / T).sum(-1).float()
    ctx = cv.cosine_verify_init(V, max_batch=B, max_draft_len=1, max_drafters=N, seed=9)
    y = torch.empty(B, dtype=torch.int32, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    cv.cosine_sample_residual(ctx, rows.to(dev), nodes.to(dev), inp["request_ids"].to(dev), y, st, step=4,
                              temperature=T,
                              row_max=None if rm is None else rm.to(dev),
                              row_sumexp=None if rs is None else rs.to(dev),
                              draft_rows=drafts.to(dev) if with_draft else None,
                              weights=wts.to(dev) if with_draft else None,
                              draft_norm=norms.to(dev) if with_draft else None)
    torch.cuda.synchronize()
    r = oracle.sample_residual(rows, nodes.numpy().astype(np.uint32), inp["request_ids"], seed=9, step=4,
                               temperature=T, row_max=rm, row_sumexp=rs, draft=drafts if with_draft else None,
                               weights=wts if with_draft else None, draft_norm=norms if with_draft else None,
                               vocab=V)
    cv.cosine_verify_destroy(ctx)
    flagged = r["tie_margin"] < 1e-6
    yy = y.cpu().numpy()
    assert not ((yy != r["out_token"]) & ~flagged).any()
    np.testing.assert_array_equal(st.cpu().numpy() & 0xff, r["status"] & 0xff)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_sample_residual_degenerate_fallback(cuda_ok, dtype):
    # q == o exactly (reading #11): a two-point target o = (1/2, 1/2) at tokens 3 and V - 5 and
    # drafter rows carrying the same two masses (two drafters, weights 1/2 each): the residual has no
    # mass on either side, the draw falls back to o over the whole row and is flagged DEGENERATE
    import paper_2503_10325_b200 as cv
    B, N, V = 48, 2, 20001
    dev = torch.device("cuda", 0)
    ld = (V + 7) // 8 * 8
    rows = torch.full((B, ld), float("-inf"), dtype=dtype)
    rows[:, 3] = 0.0
    rows[:, V - 5] = 0.0
    rows[:, V:] = float("nan")
    drafts = torch.zeros(B, N, ld, dtype=dtype)
    drafts[:, :, 3] = 0.5
    drafts[:, :, V - 5] = 0.5
    drafts[:, :, V:] = float("nan")
    wts = torch.full((B, N), 0.5)
    norms = torch.ones(B, N)
    nodes = torch.arange(B, dtype=torch.int32) % 5
    rid = torch.arange(1000, 1000 + B, dtype=torch.int64)
    ctx = cv.cosine_verify_init(V, max_batch=B, max_draft_len=1, max_drafters=N, seed=13, target_dtype=dtype,
                                draft_dtype=dtype)
    y = torch.empty(B, dtype=torch.int32, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    cv.cosine_sample_residual(ctx, rows.to(dev), nodes.to(dev), rid.to(dev), y, st, step=1,
                              draft_rows=drafts.to(dev), weights=wts.to(dev), draft_norm=norms.to(dev))
    torch.cuda.synchronize()
    cv.cosine_verify_destroy(ctx)
    r = oracle.sample_residual(rows, nodes.numpy().astype(np.uint32), rid, seed=13, step=1, draft=drafts,
                               weights=wts, draft_norm=norms, vocab=V)
    assert (r["status"] & oracle.INFO_DEGENERATE).all()
    np.testing.assert_array_equal(y.cpu().numpy(), r["out_token"])
    assert ((st.cpu().numpy() & cv.INFO_DEGENERATE) != 0).all()
    assert set(np.unique(r["out_token"])) <= {3, V - 5}
