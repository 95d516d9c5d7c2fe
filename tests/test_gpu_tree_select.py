"""TreeSelection through cosine_tree_select against orc_tree_select: tree
structure and tokens bit-exact (scores within fp32 rounding; exact ties excluded by using
distinct random confidences), and the selected tree runs through cosine_verify_tree."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _gpu(X, C, budget):
    import paper_2503_10325_b200 as cv
    dev = torch.device("cuda", 0)
    B = X.shape[0]
    ctx = cv.cosine_verify_init(1000, max_batch=B, max_draft_len=1, max_drafters=1)
    out = dict(n_nodes=torch.empty(B, dtype=torch.int32, device=dev),
               parent=torch.empty(B, budget + 1, dtype=torch.int32, device=dev),
               token=torch.empty(B, budget + 1, dtype=torch.int32, device=dev),
               score=torch.empty(B, budget + 1, dtype=torch.float32, device=dev),
               depth=torch.empty(B, budget + 1, dtype=torch.int32, device=dev))
    cv.cosine_tree_select(ctx, X.to(dev), C.to(dev), budget, out["n_nodes"], out["parent"], out["token"],
                          out["score"], out["depth"])
    torch.cuda.synchronize()
    cv.cosine_verify_destroy(ctx)
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("S,K,vocab,budget", [(8, 8, 6, 40), (8, 8, 50, 64), (2, 5, 3, 3), (16, 8, 4, 200)])
def test_tree_select_matches_oracle(cuda_ok, S, K, vocab, budget):
    g = torch.Generator().manual_seed(S * 100 + K + vocab)
    B = 64
    X = torch.randint(0, vocab, (B, S, K), generator=g, dtype=torch.int32)
    X[3, 1, 4:] = -1                      # a shorter branch
    C = torch.rand(B, S, K, generator=g) * 0.9 + 0.05
    r = oracle.tree_select(X, C.double(), budget)
    o = _gpu(X, C, budget)
    # near ties: the GPU ranks fp32 products of confidences, the oracle fp64 ones.  A request is
    # flagged when two nodes adjacent in the oracle's full ranking (budget = every node) have
    # scores within 2e-6 relative (> K fp32 roundings); its order may legitimately differ
    full = oracle.tree_select(X, C.double(), S * K)
    flagged = np.zeros(B, bool)
    for b in range(B):
        sc = np.sort(full["score"][b, 1:full["n_nodes"][b]])[::-1]
        if sc.size > 1 and (np.abs(np.diff(sc)) <= 2e-6 * sc[1:]).any():
            flagged[b] = True
    assert flagged.sum() <= max(1, 0.05 * B), flagged.sum()
    np.testing.assert_array_equal(o["n_nodes"], r["n_nodes"])
    ok = ~flagged
    np.testing.assert_array_equal(o["parent"][ok], r["parent"][ok])
    np.testing.assert_array_equal(o["token"][ok], r["token"][ok])
    np.testing.assert_array_equal(o["depth"][ok], r["depth"][ok])
    np.testing.assert_allclose(o["score"][ok], r["score"][ok], rtol=1e-6)
