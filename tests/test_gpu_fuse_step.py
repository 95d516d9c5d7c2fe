"""Drafter-side Fuse of one iteration through cosine_fuse_step against
orc_fuse_step: own tokens and the fused token bit-exact (unless the oracle's confidence gap is
a near tie), confidences within 1e-5 relative."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _gpu(logits, V, T):
    import paper_2503_10325_b200 as cv
    B, N, ld = logits.shape
    dev = torch.device("cuda", 0)
    ctx = cv.cosine_verify_init(V, max_batch=B, max_draft_len=max(1, N), max_drafters=min(N, 8),
                                draft_dtype=logits.dtype)
    x = logits.to(dev)
    own = torch.empty(B, N, dtype=torch.int32, device=dev)
    conf = torch.empty(B, N, dtype=torch.float32, device=dev)
    fused = torch.empty(B, dtype=torch.int32, device=dev)
    win = torch.empty(B, dtype=torch.int32, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    cv.cosine_fuse_step(ctx, x, own, conf, fused, win, st, temperature=T)
    torch.cuda.synchronize()
    n = cv.cosine_last_launch_count(ctx)
    cv.cosine_verify_destroy(ctx)
    return dict(own_tokens=own.cpu().numpy(), conf=conf.cpu().numpy(), fused_token=fused.cpu().numpy(),
                winner=win.cpu().numpy(), status=st.cpu().numpy(), launches=n)


def _logits(B, N, V, dtype, seed, sigma=5.0):
    g = torch.Generator().manual_seed(seed)
    ld = (V + 7) // 8 * 8
    x = torch.full((B, N, ld), float("nan"), dtype=dtype)
    x[..., :V] = (sigma * torch.randn(B, N, V, generator=g)).to(dtype)
    return x


@pytest.mark.parametrize("B,N,V,dtype,T", [(64, 4, 32000, torch.bfloat16, 1.0), (33, 3, 4099, torch.float32, 0.7),
                                         (256, 4, 128256, torch.bfloat16, 1.0), (5, 1, 9, torch.float32, 1.3)])
def test_fuse_step_matches_oracle(cuda_ok, B, N, V, dtype, T):
    x = _logits(B, N, V, dtype, seed=V + N)
    g = _gpu(x, V, T)
    r = oracle.fuse_step(x[..., :V], temperature=T)
    assert g["launches"] == 2
    np.testing.assert_array_equal(g["status"], r["status"])
    np.testing.assert_array_equal(g["own_tokens"], r["own_tokens"])  # argmax: exact (same bf16 values)
    np.testing.assert_allclose(g["conf"], r["conf"], rtol=1e-5)
    tie = r["conf_gap"] < 1e-6
    assert ((g["winner"] == r["winner"]) | tie).all()
    assert ((g["fused_token"] == r["fused_token"]) | tie).all()


def test_fuse_step_ties_and_errors(cuda_ok):
    V = 1000
    x = _logits(6, 3, V, torch.float32, seed=1, sigma=2.0)
    x[0, 1] = x[0, 0]                     # identical drafters: the tie goes to the lowest n
    x[0, 2, :V] = x[0, 0, :V] - 1.0       # same distribution again (shifted logits)
    x[1, 0, [10, 20]] = 50.0              # argmax tie inside a row: lowest index
    x[2, 2, 5] = float("nan")
    x[3, 1, :V] = float("-inf")
    x[4, 0, 7] = float("inf")
    g = _gpu(x, V, 1.0)
    r = oracle.fuse_step(x[..., :V], temperature=1.0)
    np.testing.assert_array_equal(g["status"], r["status"])
    assert list(g["status"]) == [0, 0, 3, 4, 3, 0]
    assert g["own_tokens"][1, 0] == 10
    ok = r["status"] == 0
    np.testing.assert_array_equal(g["own_tokens"][ok], r["own_tokens"][ok])
    assert g["winner"][0] in (0, 2) and r["winner"][0] in (0, 2)
