"""B200-native batched verification step of CoSine (arXiv 2503.10325).

The product path is libcosine_verify.so (hand-written sm_100a CUDA behind a C ABI,
include/cosine_verify.h); `_lib` is its ctypes binding (same names as the C entry
points) and `Verifier` a convenience owner of a context plus output buffers.
Importing this package fails loudly if the shared library is missing.
"""
from __future__ import annotations

import torch

from . import _lib
from ._lib import (  # noqa: F401
    BF16, F32, DRAFT_LOGITS, DRAFT_PROBS, INFO_DEGENERATE, INFO_NEAR_TIE, SEL_ARGMAX, SEL_SAMPLE,
    W_CONF, W_POINT, W_UNIFORM, W_WINNER, Context, CosineError, cosine_fuse_drafts,
    cosine_last_launch_count, cosine_profile_enable, cosine_profile_read,
    cosine_sample_residual,
    cosine_fuse_step, cosine_nccl_unique_id, cosine_route_update, cosine_tree_select, cosine_verify_batch, cosine_verify_batch_lazy,
    cosine_verify_destroy,
    cosine_verify_init,
    cosine_verify_tree,
    cosine_verify_init_vgroup,
    cosine_verify_batch_vgroup,
    cosine_exchange_mode,
)

__all__ = [
    "Verifier", "cosine_verify_init", "cosine_verify_destroy", "cosine_fuse_drafts",
    "cosine_verify_batch", "cosine_sample_residual", "cosine_verify_tree", "cosine_last_launch_count",
    "cosine_nccl_unique_id", "cosine_verify_batch_lazy", "cosine_fuse_step",
    "cosine_route_update", "cosine_tree_select", "cosine_verify_init_vgroup", "cosine_verify_batch_vgroup",
    "CosineError",
    "W_CONF", "W_WINNER", "W_UNIFORM", "W_POINT", "SEL_ARGMAX", "SEL_SAMPLE", "DRAFT_PROBS",
    "DRAFT_LOGITS",
]


class Verifier:
    """Owns one context and the per-call output buffers for a fixed (max) batch shape."""

    def __init__(self, vocab_size: int, *, max_batch: int, k: int, N: int, device: int = 0,
                 target_dtype=torch.bfloat16, draft_dtype=torch.bfloat16, draft_kind=DRAFT_PROBS,
                 seed: int = 0, cluster_size: int = 0, debug: bool = False, ctx=None):
        """ctx: an existing context to adopt (e.g. sharding.init_vocab_sharded's)."""
        self.V, self.k, self.N, self.device = vocab_size, k, N, device
        self.ctx = ctx if ctx is not None else cosine_verify_init(
            vocab_size, device=device, max_batch=max_batch, max_draft_len=k, max_drafters=N,
            target_dtype=target_dtype, draft_dtype=draft_dtype, draft_kind=draft_kind, seed=seed,
            cluster_size=cluster_size)
        dev = torch.device("cuda", device)
        self.accept_len = torch.empty(max_batch, dtype=torch.int32, device=dev)
        self.out_tokens = torch.empty(max_batch, k + 1, dtype=torch.int32, device=dev)
        self.status = torch.empty(max_batch, dtype=torch.int32, device=dev)
        self.debug = None
        if debug:
            f = dict(dtype=torch.float32, device=dev)
            self.debug = dict(
                p_x=torch.empty(max_batch, k, **f), q_x=torch.empty(max_batch, k, **f),
                accept_u=torch.empty(max_batch, k, **f), row_max=torch.empty(max_batch, k + 1, **f),
                row_sumexp=torch.empty(max_batch, k + 1, **f),
                draft_norm=torch.empty(max_batch, k, N, **f), conf=torch.empty(max_batch, k, N, **f),
                weights=torch.empty(max_batch, k, N, **f),
                fused_tokens=torch.empty(max_batch, k, dtype=torch.int32, device=dev),
                residual_mass=torch.empty(max_batch, **f), tie_margin=torch.empty(max_batch, **f))

    def verify(self, target, draft, draft_tokens, request_ids, *, temperature=1.0, draft_len=None,
               step=0, weight_mode=W_CONF, select_mode=SEL_ARGMAX, stream=None, lazy=False):
        """Device-resident inputs -> (accept_len, out_tokens, status) views (device).
        lazy=True: early-exit verification (cosine_verify_batch_lazy, ARGMAX only)."""
        B = target.shape[0]
        dbg = None if self.debug is None else {n: t[:B] for n, t in self.debug.items()}
        if lazy:
            if select_mode != SEL_ARGMAX:
                raise ValueError("lazy verification takes ARGMAX selection")
            cosine_verify_batch_lazy(self.ctx, target, draft, draft_tokens, request_ids,
                                     self.accept_len[:B], self.out_tokens[:B], self.status[:B],
                                     temperature=temperature, draft_len=draft_len, step=step,
                                     weight_mode=weight_mode, debug=dbg, stream=stream)
        else:
            cosine_verify_batch(self.ctx, target, draft, draft_tokens, request_ids,
                                self.accept_len[:B], self.out_tokens[:B], self.status[:B],
                                temperature=temperature, draft_len=draft_len, step=step,
                                weight_mode=weight_mode, select_mode=select_mode, debug=dbg,
                                stream=stream)
        return self.accept_len[:B], self.out_tokens[:B], self.status[:B]

    def verify_host(self, host_inputs: dict, dev_buffers: dict, *, temperature=1.0, step=0,
                    weight_mode=W_CONF, select_mode=SEL_ARGMAX, stream=None):
        """End-to-end call from (pinned) host tensors: H2D copies into `dev_buffers`, the kernel
        and the D2H read of the results, all on ONE stream (`stream`, default the current one),
        which is synchronized before returning.  Returns host (accept_len, out_tokens, status),
        valid on return (pinned buffers owned by this Verifier, overwritten by the next call)."""
        s = stream if stream is not None else torch.cuda.current_stream(torch.device("cuda", self.device))
        with torch.cuda.stream(s):
            for name in ("target", "draft", "draft_tokens", "request_ids"):
                dev_buffers[name].copy_(host_inputs[name], non_blocking=True)
            dl = None
            if host_inputs.get("draft_len") is not None:
                dev_buffers["draft_len"].copy_(host_inputs["draft_len"], non_blocking=True)
                dl = dev_buffers["draft_len"]
            a, o, st = self.verify(dev_buffers["target"], dev_buffers["draft"], dev_buffers["draft_tokens"],
                                   dev_buffers["request_ids"], temperature=temperature, draft_len=dl,
                                   step=step, weight_mode=weight_mode, select_mode=select_mode, stream=s)
            B = a.shape[0]
            if getattr(self, "_host_out", None) is None or self._host_out[0].shape[0] < B:
                self._host_out = tuple(torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (a, o, st))
            out = tuple(h[:B] for h in self._host_out)
            for h, d in zip(out, (a, o, st)):
                h.copy_(d, non_blocking=True)
        s.synchronize()
        return out

    def close(self):
        if self.ctx is not None:
            cosine_verify_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
