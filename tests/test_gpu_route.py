"""Routing feedback through cosine_route_update against orc_route_update:
routing scores and draft accuracies within 1e-5, statuses exact; the verification outputs feed it
(accept_len / out_tokens of cosine_verify_batch as the accepted tokens)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _gpu(X, c, acc, L, E, M, part=None, decay=0.9):
    import paper_2503_10325_b200 as cv
    dev = torch.device("cuda", 0)
    B, N, K = X.shape
    ctx = cv.cosine_verify_init(E.shape[0], max_batch=B, max_draft_len=K, max_drafters=min(N, 8))
    Mg = M.clone().float().to(dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    d = torch.empty(B, N, K, dtype=torch.float32, device=dev)
    cv.cosine_route_update(ctx, X.to(dev), c.float().to(dev), acc.to(dev), L.to(dev), E.to(dev), Mg, st,
                           participating=None if part is None else part.to(dev), decay=decay, d_out=d)
    torch.cuda.synchronize()
    cv.cosine_verify_destroy(ctx)
    return Mg.cpu().numpy(), d.cpu().numpy(), st.cpu().numpy()


@pytest.mark.parametrize("dtype,H", [(torch.bfloat16, 4096), (torch.float32, 264)])
def test_route_update_matches_oracle(cuda_ok, dtype, H):
    g = torch.Generator().manual_seed(H)
    B, N, K, V = 48, 4, 8, 5003
    E = torch.randn(V, H, generator=g).to(dtype)
    acc = torch.randint(0, V, (B, K + 1), generator=g, dtype=torch.int32)
    X = torch.randint(0, V, (B, N, K), generator=g, dtype=torch.int32)
    X[:, 0, :] = acc[:, :K]                      # node 0 drafted the accepted tokens (d = 1)
    X[:, 1, :4] = acc[:, :4]
    L = torch.randint(-1, K + 1, (B,), generator=g, dtype=torch.int32)
    c = torch.rand(B, N, K, generator=g)
    M = torch.rand(B, N, generator=g)
    part = (torch.rand(B, N, generator=g) > 0.2).to(torch.uint8)
    X[5, 2, 3] = V + 1                           # a bad token -> status 2, M kept
    L[5] = 4
    Mg, dg, st = _gpu(X, c, acc, L, E, M, part=part)
    r = oracle.route_update(X, c.float().double(), acc, L, E, M.float().double(), participating=part)
    np.testing.assert_array_equal(st, r["status"])
    assert st[5] == 2
    np.testing.assert_allclose(Mg, r["M"], rtol=1e-5, atol=1e-6)
    ok = (L.numpy() >= 0) & (st == 0)
    mask = ok[:, None, None] & (part.numpy()[:, :, None] != 0)
    np.testing.assert_allclose(dg[np.broadcast_to(mask, dg.shape)], r["d"][np.broadcast_to(mask, dg.shape)],
                               rtol=1e-5, atol=1e-5)


def test_route_update_after_verification(cuda_ok):
    # the post-verification step of Alg. 1: out_tokens / accept_len of cosine_verify_batch
    import synth
    from tests import parity
    B, k, N, V = 32, 6, 3, 3001
    inp = synth.linear_inputs(B, k, N, V, dtype=torch.bfloat16, seed=11)
    out = parity.gpu_verify(inp)
    X = inp["draft_tokens"].permute(0, 2, 1).contiguous()       # [B][N][k] node-major
    c = torch.rand(B, N, k, generator=torch.Generator().manual_seed(2))
    E = torch.randn(V, 1024, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16)
    acc = torch.as_tensor(out["out_tokens"])
    L = torch.as_tensor(out["accept_len"])
    M = torch.full((B, N), 0.5)
    Mg, _, st = _gpu(X, c, acc, L, E, M)
    r = oracle.route_update(X, c.double(), acc, L, E, M.double())
    np.testing.assert_array_equal(st, r["status"])
    np.testing.assert_allclose(Mg, r["M"], rtol=1e-5, atol=1e-6)
