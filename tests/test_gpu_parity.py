"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs.  Accept lengths, emitted tokens and statuses are bit-exact except where the oracle
flags a near tie (margin < 1e-6, north_star); probabilities within 1e-5 relative."""
import numpy as np
import pytest
import torch

import synth

from . import parity

pytestmark = pytest.mark.gpu

W_CONF, W_WINNER, W_UNIFORM, W_POINT = 0, 1, 2, 3


def _run(inp, name="", **kw):
    subset = kw.pop("subset", None)
    g = parity.gpu_verify(inp, **kw)
    kw.pop("cluster_size", None)
    r = parity.oracle_verify(inp, subset=subset, **kw)
    frac = parity.MAX_FLAG_FRAC_SAMPLE if kw.get("sm", 0) == 1 else parity.MAX_FLAG_FRAC
    return g, r, parity.compare(g, r, subset=subset, greedy=kw.get("T", 1.0) == 0.0, name=name, max_flag_frac=frac)


def test_c1_full(cuda_ok):
    c = synth.CONFIGS["c1"]
    inp = synth.linear_inputs(c["B"], c["k"], c["N"], c["V"], dtype=c["dtype"], seed=11)
    g, r, _ = _run(inp, name="c1")
    assert (g["status"] & 0xff == 0).all()


def test_c2_full(cuda_ok):
    c = synth.CONFIGS["c2"]
    inp = synth.linear_inputs(c["B"], c["k"], c["N"], c["V"], dtype=c["dtype"], seed=12, device="cuda")
    g, r, (mism, flagged) = _run(inp, name="c2")
    assert g["accept_len"].min() >= 0


@pytest.mark.parametrize("V,dtype", [(5, torch.float32), (8, torch.bfloat16), (9, torch.float32),
                                     (1003, torch.float32), (2051, torch.bfloat16), (4097, torch.bfloat16)])
def test_ragged_vocab(cuda_ok, V, dtype):
    # partial last group, chunks spanning several tiles, NaN padding past V must never be read
    inp = synth.linear_inputs(24, 5, 3, V, dtype=dtype, seed=V, sigma=2.0, draft_len="random")
    _run(inp)


@pytest.mark.parametrize("wm,sm", [(W_CONF, 0), (W_WINNER, 0), (W_UNIFORM, 0), (W_POINT, 0),
                                   (W_CONF, 1), (W_WINNER, 1), (W_UNIFORM, 1)])
def test_weight_and_select_modes(cuda_ok, wm, sm):
    inp = synth.linear_inputs(32, 6, 3, 7000, dtype=torch.bfloat16, seed=100 + wm + 10 * sm)
    _run(inp, wm=wm, sm=sm)


def test_greedy(cuda_ok):
    inp = synth.linear_inputs(48, 8, 4, 32000, dtype=torch.bfloat16, seed=21, token_mode="argmax",
                              draft_len="random")
    g, r, (mism, flagged) = _run(inp, T=0.0)
    assert mism == 0  # greedy decisions compare exact bf16 values: no ties to flag


@pytest.mark.parametrize("T", [0.7, 1.3])
def test_logits_drafts_and_temperature(cuda_ok, T):
    inp = synth.linear_inputs(16, 4, 2, 5000, dtype=torch.float32, seed=31, draft_kind="logits")
    _run(inp, T=T, draft_kind="logits")


def test_mixed_dtypes(cuda_ok):
    inp = synth.linear_inputs(16, 4, 3, 6000, dtype=torch.float32, draft_dtype=torch.bfloat16, seed=41)
    _run(inp)


@pytest.mark.parametrize("cs", [1, 2, 4, 8, 16])
def test_chunking_invariance(cuda_ok, cs):
    inp = synth.linear_inputs(16, 6, 4, 20000, dtype=torch.bfloat16, seed=51)
    _run(inp, cluster_size=cs)


def test_draft_equals_target_accepts_all(cuda_ok):
    # q = o  =>  min(1, o/q) = 1: identical logits rows, N = 1, LOGITS drafts
    inp = synth.linear_inputs(64, 8, 1, 32000, dtype=torch.bfloat16, seed=61, rho_hi=1.0, rho_lo=1.0,
                              draft_kind="logits")
    assert torch.equal(inp["draft"][:, :, 0, :32000], inp["target"][:, :8, :32000])
    g = parity.gpu_verify(inp, draft_kind="logits")
    assert (g["accept_len"] == 8).all()
    np.testing.assert_array_equal(g["out_tokens"][:, :8], inp["draft_tokens"][:, :, 0].numpy())


def test_errors_are_per_request(cuda_ok):
    inp = synth.linear_inputs(8, 3, 2, 3000, dtype=torch.float32, seed=71)
    t, d, X = inp["target"], inp["draft"], inp["draft_tokens"]
    d[1, 0, 1, X[1, 0, 1]] = 0.0          # zero-probability own token
    X[2, 1, 0] = 3000                      # out of range
    t[3, 2, 17] = float("nan")             # NaN logit
    d[4, 1, 0, 5] = -0.25                  # negative probability
    t[5, 0, :3000] = float("-inf")         # empty row
    inp["draft_len"] = torch.full((8,), 3, dtype=torch.int32)
    inp["draft_len"][6] = 0                # bad gamma
    g = parity.gpu_verify(inp)
    r = parity.oracle_verify(inp)
    np.testing.assert_array_equal(g["status"] & 0xff, r["status"] & 0xff)
    assert list(r["status"][:7] & 0xff) == [0, 1, 2, 3, 3, 4, 5]
    np.testing.assert_array_equal(g["accept_len"][1:7], -1)
    parity.compare(g, r, check_probs=False)


def test_rows_past_draft_len_never_read(cuda_ok):
    inp = synth.linear_inputs(12, 6, 3, 5000, dtype=torch.bfloat16, seed=81, draft_len="random")
    g1 = parity.gpu_verify(inp)
    for b in range(12):
        gb = int(inp["draft_len"][b])
        inp["target"][b, gb + 1:] = float("nan")
        inp["draft"][b, gb:] = float("nan")
    g2 = parity.gpu_verify(inp)
    np.testing.assert_array_equal(g1["out_tokens"], g2["out_tokens"])
    assert (g2["status"] & 0xff == 0).all()


def test_batch_order_and_repeat_invariance(cuda_ok):
    # reading #8: results depend on global request ids only
    inp = synth.linear_inputs(40, 6, 3, 9000, dtype=torch.bfloat16, seed=91)
    g1 = parity.gpu_verify(inp)
    g1b = parity.gpu_verify(inp)
    np.testing.assert_array_equal(g1["out_tokens"], g1b["out_tokens"])
    perm = torch.randperm(40, generator=torch.Generator().manual_seed(0))
    inp2 = {k: (v[perm] if torch.is_tensor(v) and v.dim() > 0 and v.shape[0] == 40 else v) for k, v in inp.items()}
    g2 = parity.gpu_verify(inp2)
    np.testing.assert_array_equal(g1["out_tokens"][perm.numpy()], g2["out_tokens"])
    # batch sharding: two halves on two contexts give the same per-request results
    h1 = {k: (v[:20] if torch.is_tensor(v) and v.dim() > 0 and v.shape[0] == 40 else v) for k, v in inp.items()}
    h2 = {k: (v[20:] if torch.is_tensor(v) and v.dim() > 0 and v.shape[0] == 40 else v) for k, v in inp.items()}
    gh = np.concatenate([parity.gpu_verify(h1)["out_tokens"], parity.gpu_verify(h2)["out_tokens"]])
    np.testing.assert_array_equal(g1["out_tokens"], gh)


def test_c3_full_size_all_requests(cuda_ok):
    # BASELINE config c3 in the launch configuration bench.py times: all 256 requests
    c = synth.CONFIGS["c3"]
    inp = synth.linear_inputs(c["B"], c["k"], c["N"], c["V"], dtype=c["dtype"], seed=1234, device="cuda")
    g = parity.gpu_verify(inp)
    r = parity.oracle_verify(inp)
    parity.compare(g, r, name="c3")


@pytest.mark.parametrize("wm", [W_CONF, W_WINNER])
def test_c3_full_size_sample_select(cuda_ok, wm):
    # SAMPLE selection (x* ~ fused q, reading #3) at BASELINE config c3: every request
    c = synth.CONFIGS["c3"]
    inp = synth.linear_inputs(c["B"], c["k"], c["N"], c["V"], dtype=c["dtype"], seed=1235, device="cuda")
    _run(inp, wm=wm, sm=1, name=f"c3 SAMPLE wm={wm}")


@pytest.mark.parametrize("T", [0.7, 1.3])
def test_sample_select_logits_drafts(cuda_ok, T):
    inp = synth.linear_inputs(24, 5, 3, 6007, dtype=torch.float32, seed=37, draft_kind="logits",
                              draft_len="random")
    _run(inp, T=T, draft_kind="logits", sm=1, name=f"SAMPLE logits T={T}")


@pytest.mark.parametrize("cs", [1, 4, 16])
def test_sample_select_chunking(cuda_ok, cs):
    # the draw's crossing chunk comes from the statistics pass's chunk records: any chunking
    inp = synth.linear_inputs(16, 6, 4, 20000, dtype=torch.bfloat16, seed=52)
    _run(inp, sm=1, cluster_size=cs, name=f"SAMPLE C={cs}")


@pytest.mark.parametrize("V,dtype", [(5, torch.float32), (1003, torch.float32), (2051, torch.bfloat16),
                                     (40003, torch.bfloat16)])
def test_sample_select_ragged_tail_mass(cuda_ok, V, dtype):
    # SAMPLE draws over probability drafts locate their 32-group slice from the statistics pass;
    # the row's partial last group is in no slice.  Half of every drafter row's mass is moved
    # into the last V % 8 entries so that many draws land there (and in the last full slices)
    inp = synth.linear_inputs(32, 5, 3, V, dtype=dtype, seed=V + 7, draft_len="random")
    d = inp["draft"]
    tail = V % 8
    if V > tail:
        body = d[..., : V - tail].float()
        d[..., : V - tail] = (body / body.sum(-1, keepdim=True) * 0.5).to(dtype)
        d[..., V - tail:V] = 0.5 / tail
    else:
        d[..., :V] = 1.0 / V
    _run(inp, sm=1, name=f"SAMPLE tail V={V}")


@pytest.mark.slow
def test_gpu_output_distribution_chi_square(cuda_ok):
    # SAMPLE fusion is distribution exact (reading #3): the first emitted token ~ o_0
    import scipy.stats
    V, n = 6, 20000
    base = synth.tiny_inputs(1, 2, 3, V, seed=5)
    inp = {k: (v.expand(n, *v.shape[1:]).contiguous() if torch.is_tensor(v) and v.dim() > 1 else v)
           for k, v in base.items()}
    inp["request_ids"] = torch.arange(n, dtype=torch.int64)
    # drafter own tokens only enter the weights; keep the row's tokens
    g = parity.gpu_verify(inp, sm=1, wm=W_UNIFORM)
    p = torch.softmax(base["target"][0, 0, :V].double(), -1).numpy()
    counts = np.bincount(g["out_tokens"][:, 0], minlength=V)
    assert scipy.stats.chisquare(counts, p * n).pvalue > 1e-4


@pytest.mark.parametrize("B,k,N,V,dtype", [(1, 4, 2, 32000, torch.float32), (64, 8, 3, 32000, torch.bfloat16),
                                           (7, 5, 4, 20011, torch.bfloat16)])
def test_one_launch_small_batch_path(cuda_ok, B, k, N, V, dtype):
    # small batches run as ONE cooperative launch (tiny_kernel); a fixed chunk count forces the
    # three-launch split path.  Both against the oracle; identical outputs where nothing is flagged
    inp = synth.linear_inputs(B, k, N, V, dtype=dtype, seed=B * 31 + k, draft_len="random")
    g1, r, _ = _run(inp, name=f"one-launch B={B}")
    assert g1["launches"] == 1
    g3 = parity.gpu_verify(inp, cluster_size=4)
    assert g3["launches"] == 3
    ok = r["tie_margin"] >= parity.TIE
    np.testing.assert_array_equal(g1["accept_len"][ok], g3["accept_len"][ok])
    np.testing.assert_array_equal(g1["out_tokens"][ok], g3["out_tokens"][ok])
