"""One context across every single-GPU path in sequence: the one-launch small-batch kernel, the
three-launch split path (ARGMAX and SAMPLE), the lazy rounds, again the small path.  Each path
leaves the context's device counters clean for the next call (they are reset by the kernels that
consume them), so every call must give exactly the outputs of a fresh context on the same
inputs."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _call(ver, inp, **kw):
    a, o, s = ver.verify(inp["target"], inp["draft"], inp["draft_tokens"], inp["request_ids"],
                         draft_len=inp["draft_len"], **kw)
    torch.cuda.synchronize()
    return a.cpu().numpy().copy(), o.cpu().numpy().copy(), s.cpu().numpy().copy()


def test_context_reuse_across_paths(cuda_ok):
    import paper_2503_10325_b200 as cv
    V, k, N = 32000, 8, 3
    dev = torch.device("cuda", 0)
    inputs = {
        "small": synth.linear_inputs(8, k, N, V, dtype=torch.bfloat16, seed=901, device=dev, draft_len="random"),
        "large": synth.linear_inputs(192, k, N, V, dtype=torch.bfloat16, seed=902, device=dev, draft_len="random"),
        "mid": synth.linear_inputs(48, k, N, V, dtype=torch.bfloat16, seed=903, device=dev),
    }
    seq = [("small", {}), ("large", {}), ("large", {"select_mode": cv.SEL_SAMPLE}), ("mid", {"lazy": True}),
           ("small", {}), ("large", {}), ("mid", {}), ("large", {"select_mode": cv.SEL_SAMPLE}), ("small", {})]
    shared = cv.Verifier(V, max_batch=192, k=k, N=N, seed=5)
    launches = []
    for name, kw in seq:
        got = _call(shared, inputs[name], **kw)
        launches.append(cv.cosine_last_launch_count(shared.ctx))
        fresh = cv.Verifier(V, max_batch=192, k=k, N=N, seed=5)
        ref = _call(fresh, inputs[name], **kw)
        fresh.close()
        for g, r in zip(got, ref):
            np.testing.assert_array_equal(g, r, err_msg=f"{name} {kw}")
    shared.close()
    assert launches[0] == 1 and launches[1] == 3  # the one-launch path and the split path both ran


def test_two_contexts_on_two_streams(cuda_ok):
    # calls on different streams may overlap on the device (the one-launch kernel is a cooperative
    # launch; the split path's waits only target CTAs of its own, already started, grids)
    import paper_2503_10325_b200 as cv
    V, k, N = 32000, 8, 3
    dev = torch.device("cuda", 0)
    a_in = synth.linear_inputs(16, k, N, V, dtype=torch.bfloat16, seed=911, device=dev)
    b_in = synth.linear_inputs(160, k, N, V, dtype=torch.bfloat16, seed=912, device=dev)
    va, vb = cv.Verifier(V, max_batch=160, k=k, N=N, seed=3), cv.Verifier(V, max_batch=160, k=k, N=N, seed=3)
    ref_a, ref_b = _call(va, a_in), _call(vb, b_in)
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    for _ in range(20):
        for ver, inp, s in ((va, a_in, sa), (vb, b_in, sb)):
            ver.verify(inp["target"], inp["draft"], inp["draft_tokens"], inp["request_ids"], stream=s)
    torch.cuda.synchronize()
    for ver, ref in ((va, ref_a), (vb, ref_b)):
        B = ref[0].shape[0]
        np.testing.assert_array_equal(ver.accept_len[:B].cpu().numpy(), ref[0])
        np.testing.assert_array_equal(ver.out_tokens[:B].cpu().numpy(), ref[1])
    va.close()
    vb.close()
