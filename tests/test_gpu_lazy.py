"""Lazy / early-exit verification through cosine_verify_batch_lazy: the
outputs must equal the full parallel verification's (and the oracle's) on valid inputs, with
2 ceil((k+1)/2) + 1 launches; a data error in a row after the first rejection is, by design, not seen."""
import numpy as np
import pytest
import torch

import synth
from paper_2503_10325_b200 import W_CONF, W_POINT, W_WINNER
from tests import parity


def _same(a, b):
    assert (a["accept_len"] == b["accept_len"]).all()
    assert (a["out_tokens"] == b["out_tokens"]).all()
    assert ((a["status"] & 0xff) == (b["status"] & 0xff)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    dict(B=64, k=8, N=3, V=32000, dtype=torch.bfloat16, T=1.0, wm=W_CONF),
    dict(B=40, k=6, N=4, V=4099, dtype=torch.bfloat16, T=1.0, wm=W_WINNER, draft_len="random"),
    dict(B=32, k=4, N=2, V=2053, dtype=torch.bfloat16, T=1.0, wm=W_POINT),
    dict(B=32, k=5, N=3, V=3001, dtype=torch.bfloat16, T=0.0, wm=W_CONF),
    dict(B=24, k=4, N=3, V=2051, dtype=torch.float32, T=0.7, wm=W_CONF, draft_kind="logits"),
])
def test_lazy_equals_full_and_oracle(cuda_ok, case):
    c = dict(case)
    T, wm, dk = c.pop("T"), c.pop("wm"), c.pop("draft_kind", "probs")
    dl = c.pop("draft_len", None)
    inp = synth.linear_inputs(c["B"], c["k"], c["N"], c["V"], dtype=c["dtype"], seed=77, draft_len=dl,
                              draft_kind=dk)
    full = parity.gpu_verify(inp, T=T, wm=wm, draft_kind=dk)
    lazy = parity.gpu_verify(inp, T=T, wm=wm, draft_kind=dk, lazy=True)
    _same(lazy, full)
    assert lazy["launches"] == 2 * ((c["k"] + 2) // 2) + 1  # 2 positions per round + the final draws
    r = parity.oracle_verify(inp, T=T, wm=wm, draft_kind=dk)
    parity.compare(lazy, r, check_probs=False, greedy=(T == 0.0))


@pytest.mark.gpu
def test_lazy_c3_full_size(cuda_ok):
    cfg = synth.CONFIGS["c3"]
    inp = synth.linear_inputs(cfg["B"], cfg["k"], cfg["N"], cfg["V"], dtype=cfg["dtype"], seed=1234,
                              device="cuda")
    full = parity.gpu_verify(inp)
    lazy = parity.gpu_verify(inp, lazy=True)
    _same(lazy, full)
    r = parity.oracle_verify(inp)  # every request
    parity.compare(lazy, r, check_probs=False, name="c3 lazy")


@pytest.mark.gpu
def test_lazy_does_not_read_rows_after_the_stop(cuda_ok):
    inp = synth.linear_inputs(32, 6, 3, 3001, dtype=torch.bfloat16, seed=5)
    clean = parity.gpu_verify(inp)
    # poison every row after each request's first rejection (NaN): the full path reports the
    # error, the lazy path never reads those rows and returns the clean result
    bad = {k: (v.clone() if torch.is_tensor(v) else v) for k, v in inp.items()}
    poisoned = []
    for b in range(32):
        L = int(clean["accept_len"][b])
        if L + 1 <= 6:
            bad["target"][b, L + 1:, :5] = float("nan")
            bad["draft"][b, L + 1:, :, :5] = float("nan")
            poisoned.append(b)
    assert poisoned
    full = parity.gpu_verify(bad)
    lazy = parity.gpu_verify(bad, lazy=True)
    _same(lazy, clean)
    assert (full["status"][poisoned] & 0xff != 0).all()
