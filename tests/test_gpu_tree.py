"""GPU parity of cosine_verify_tree (reading #13) against orc_verify_tree."""
import numpy as np
import pytest
import torch

import oracle
import synth

from . import parity

pytestmark = pytest.mark.gpu


def _gpu_tree(t, *, seed=3, step=0, wm=0, T=1.0, dtype=torch.float32, lazy=False):
    import paper_2503_10325_b200 as cv
    dev = torch.device("cuda", 0)
    B, nn, _ = t["target"].shape
    N = t["draft"].shape[2]
    ctx = cv.cosine_verify_init(t["V"], max_batch=B, max_draft_len=1, max_drafters=N, seed=seed,
                                target_dtype=t["target"].dtype, draft_dtype=t["draft"].dtype,
                                max_tree_nodes=nn)
    al = torch.empty(B, dtype=torch.int32, device=dev)
    an = torch.empty(B, nn, dtype=torch.int32, device=dev)
    ot = torch.empty(B, nn, dtype=torch.int32, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    d = {k: (v.to(dev) if torch.is_tensor(v) else v) for k, v in t.items()}
    cv.cosine_verify_tree(ctx, d["parent"], d["node_token"], d["internal_row"], d["target"], d["draft"],
                          d["node_draft_tokens"], d["request_ids"], al, an, ot, st, temperature=T, step=step,
                          weight_mode=wm, lazy=lazy)
    torch.cuda.synchronize()
    launches = cv.cosine_last_launch_count(ctx)
    cv.cosine_verify_destroy(ctx)
    return dict(accept_len=al.cpu().numpy(), accepted_nodes=an.cpu().numpy(), out_tokens=ot.cpu().numpy(),
                status=st.cpu().numpy(), launches=launches)


def _oracle_tree(t, *, seed=3, step=0, wm=0, T=1.0, subset=None):
    """orc_verify_tree, one request per host thread task (oracle.by_request)."""
    sel = slice(None) if subset is None else subset
    args = [t[n][sel].cpu() for n in ("parent", "node_token", "internal_row", "target", "draft",
                                      "node_draft_tokens", "request_ids")]
    return oracle.by_request(lambda *a: oracle.verify_tree(*a, temperature=T, seed=seed, step=step, weight_mode=wm,
                                                           vocab=t["V"]), *args)


def _compare(g, r, subset=None, name="tree"):
    idx = np.arange(len(r["accept_len"])) if subset is None else np.asarray(subset)
    np.testing.assert_array_equal(g["status"][idx] & 0xff, r["status"] & 0xff)
    mism = (g["accept_len"][idx] != r["accept_len"]) | (g["out_tokens"][idx] != r["out_tokens"]).any(1) | \
           (g["accepted_nodes"][idx] != r["accepted_nodes"]).any(1)
    flagged = r["tie_margin"] < 1e-6
    parity.record(name, requests=int(len(idx)), mismatches=int(mism.sum()),
                  unflagged_mismatches=int((mism & ~flagged).sum()), flagged=int(flagged.sum()))
    assert not (mism & ~flagged).any(), np.nonzero(mism & ~flagged)[0][:5]
    assert flagged.sum() <= max(1, parity.MAX_FLAG_FRAC * len(idx))
    return int(mism.sum()), int(flagged.sum())


@pytest.mark.parametrize("lazy", [False, True])
@pytest.mark.parametrize("schedule,cap,V,wm", [((2, 2, 1), 12, 1003, 0), ((3, 1, 1, 1), 20, 777, 1),
                                               ((4, 2, 2, 1, 1, 1, 1, 1), 64, 2049, 2)])
def test_tree_small(cuda_ok, schedule, cap, V, wm, lazy):
    t = synth.tree_inputs(24, 3, V, schedule=schedule, cap=cap, dtype=torch.float32, seed=V, sigma=2.0)
    g = _gpu_tree(t, wm=wm, step=1, lazy=lazy)
    r = _oracle_tree(t, wm=wm, step=1)
    _compare(g, r)
    assert g["launches"] == (1 if lazy else 3)


def test_chain_tree_equals_linear_on_gpu(cuda_ok):
    # a chain tree is the linear path (same Philox stream), here on the GPU
    from . import parity
    inp = synth.linear_inputs(32, 5, 2, 3001, dtype=torch.float32, seed=7, sigma=3.0)
    g_lin = parity.gpu_verify(inp, seed=21)
    B, k = 32, 5
    t = dict(parent=torch.arange(-1, k, dtype=torch.int32).expand(B, k + 1).contiguous(),
             node_token=torch.cat([torch.zeros(B, 1, dtype=torch.int32),
                                   torch.as_tensor(g_lin["fused_tokens"])], 1).contiguous(),
             internal_row=torch.tensor(list(range(k)) + [-1], dtype=torch.int32).expand(B, k + 1).contiguous(),
             target=inp["target"], draft=inp["draft"], node_draft_tokens=inp["draft_tokens"],
             request_ids=inp["request_ids"], V=inp["V"])
    for lazy in (False, True):
        g_tree = _gpu_tree(t, seed=21, lazy=lazy)
        np.testing.assert_array_equal(g_tree["accept_len"], g_lin["accept_len"])
        np.testing.assert_array_equal(g_tree["out_tokens"], g_lin["out_tokens"])


def test_bad_tree_and_errors(cuda_ok):
    t = synth.tree_inputs(6, 2, 500, schedule=(2, 1), cap=6, dtype=torch.float32, seed=9, sigma=2.0)
    t["parent"][1, 3] = 5                      # parent after child
    t["node_token"][2, 2] = t["node_token"][2, 1]  # duplicate sibling token
    t["node_token"][3, 4] = 500                # token out of range
    t["target"][4, 2, 7] = float("nan")        # non-finite logit
    g = _gpu_tree(t)
    r = _oracle_tree(t)
    np.testing.assert_array_equal(g["status"] & 0xff, r["status"] & 0xff)
    assert list(r["status"][:5] & 0xff) == [0, 6, 6, 2, 3]
    _compare(g, r)


def test_c4_full_size_all_requests(cuda_ok):
    # BASELINE config c4 (128 requests x 65 nodes, V = 128256) in the bench's launch
    # configuration: every request against the oracle
    c = synth.CONFIGS["c4"]
    t = synth.tree_inputs(c["B"], c["N"], c["V"], dtype=c["dtype"], seed=44, device="cuda")
    g = _gpu_tree(t, seed=5)
    r = _oracle_tree(t, seed=5)
    _compare(g, r, name="c4 all-nodes")


def test_lazy_tree_c4_full_size_equals_full(cuda_ok):
    # NEXT-1: the lazy walk reads only the visited nodes and must reproduce the all-nodes result
    c = synth.CONFIGS["c4"]
    t = synth.tree_inputs(c["B"], c["N"], c["V"], dtype=c["dtype"], seed=45, device="cuda")
    full = _gpu_tree(t, seed=6)
    lazy = _gpu_tree(t, seed=6, lazy=True)
    tie = ((full["status"] | lazy["status"]) & 0x200) != 0
    diff = (full["accept_len"] != lazy["accept_len"]) | (full["out_tokens"] != lazy["out_tokens"]).any(1) | \
           (full["accepted_nodes"] != lazy["accepted_nodes"]).any(1) | \
           ((full["status"] & 0xff) != (lazy["status"] & 0xff))
    assert not (diff & ~tie).any(), np.nonzero(diff & ~tie)[0][:5]
    assert lazy["launches"] == 1
    r = _oracle_tree(t, seed=6)
    _compare(lazy, r, name="c4 lazy")


def test_lazy_tree_errors(cuda_ok):
    t = synth.tree_inputs(6, 2, 500, schedule=(2, 1), cap=6, dtype=torch.float32, seed=9, sigma=2.0)
    clean = _gpu_tree(t)
    t["parent"][1, 3] = 5                      # structure errors: checked for the whole tree
    t["node_token"][2, 2] = t["node_token"][2, 1]
    t["target"][4, 0, 7] = float("nan")        # the root is always visited
    # request 5: poison a leaf the walk does not visit (reading #23: not detected)
    path5 = set(int(x) for x in clean["accepted_nodes"][5] if x >= 0) | {0}
    leaves = [j for j in range(1, t["parent"].shape[1]) if int(t["internal_row"][5, j]) < 0 and j not in path5]
    t["target"][5, leaves[0], 3] = float("nan")
    lazy = _gpu_tree(t, lazy=True)
    assert list(lazy["status"][:5] & 0xff) == [0, 6, 6, 0, 3]
    assert lazy["status"][5] & 0xff == 0
    assert lazy["accept_len"][5] == clean["accept_len"][5]
    np.testing.assert_array_equal(lazy["out_tokens"][5], clean["out_tokens"][5])
