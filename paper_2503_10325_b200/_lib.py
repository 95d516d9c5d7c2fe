"""ctypes binding of libcosine_verify.so — argument marshalling only.

Every function here has the name of the C entry point it calls
(include/cosine_verify.h) and does nothing but turn torch tensors into device
pointers / sizes and C status codes into exceptions.  Every step of the method
runs in the CUDA kernels.  There is no CPU fallback: if the shared library is
missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcosine_verify.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2503_10325_b200/build.py` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

BF16, F32 = 0, 1
DRAFT_PROBS, DRAFT_LOGITS = 0, 1
W_CONF, W_WINNER, W_UNIFORM, W_POINT = 0, 1, 2, 3
SEL_ARGMAX, SEL_SAMPLE = 0, 1
REQ_OK, REQ_ZERO_PROB, REQ_TOKEN_RANGE, REQ_NONFINITE, REQ_EMPTY, REQ_BAD_LEN = range(6)
INFO_DEGENERATE, INFO_NEAR_TIE = 0x100, 0x200
STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "UNSUPPORTED", 3: "CUDA", 4: "NCCL", 5: "OUT_OF_MEMORY"}

_P = ctypes.c_void_p
_i32, _u32, _i64, _u64, _f32 = ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float


class cosine_config_t(ctypes.Structure):
    _fields_ = [
        ("device", _i32), ("vocab_size", _i64), ("vocab_begin", _i64), ("vocab_end", _i64),
        ("max_batch", _i32), ("max_draft_len", _i32), ("max_drafters", _i32), ("max_tree_nodes", _i32),
        ("target_dtype", ctypes.c_int), ("draft_dtype", ctypes.c_int), ("draft_kind", ctypes.c_int),
        ("seed", _u64), ("nranks", _i32), ("rank", _i32), ("nccl_unique_id", _P),
        ("cluster_size", _i32), ("exchange", _i32),
    ]


class cosine_debug_t(ctypes.Structure):
    _fields_ = [(n, _P) for n in ("p_x", "q_x", "accept_u", "row_max", "row_sumexp", "draft_norm",
                                  "conf", "weights", "fused_tokens", "residual_mass", "tie_margin")]


_lib.cosine_verify_init.argtypes = [ctypes.POINTER(cosine_config_t), ctypes.POINTER(_P)]
_lib.cosine_verify_init.restype = ctypes.c_int
_lib.cosine_verify_destroy.argtypes = [_P]
_lib.cosine_verify_destroy.restype = ctypes.c_int
_lib.cosine_last_error.argtypes = [_P]
_lib.cosine_last_error.restype = ctypes.c_char_p
_lib.cosine_last_launch_count.argtypes = [_P]
_lib.cosine_last_launch_count.restype = _i32
_lib.cosine_exchange_mode.argtypes = [_P]
_lib.cosine_exchange_mode.restype = _i32
_lib.cosine_fuse_drafts.argtypes = [_P, _P, _i32, _i32, _i32, _P, _i64, _P, _P, _u32, _f32,
                                    ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _i64, _P]
_lib.cosine_fuse_drafts.restype = ctypes.c_int
_lib.cosine_verify_batch.argtypes = [_P, _P, _i32, _i32, _i32, _P, _i64, _f32, _P, _i64, _P, _P,
                                     _P, _u32, ctypes.c_int, ctypes.c_int, _P, _P, _P,
                                     ctypes.POINTER(cosine_debug_t)]
_lib.cosine_verify_batch.restype = ctypes.c_int
_lib.cosine_verify_batch_lazy.argtypes = [_P, _P, _i32, _i32, _i32, _P, _i64, _f32, _P, _i64, _P, _P,
                                          _P, _u32, ctypes.c_int, _P, _P, _P,
                                          ctypes.POINTER(cosine_debug_t)]
_lib.cosine_verify_batch_lazy.restype = ctypes.c_int
_lib.cosine_sample_residual.argtypes = [_P, _P, _i32, _P, _i64, _f32, _P, _P, _P, _i64, _P, _P,
                                        _i32, _P, _P, _u32, _P, _P]
_lib.cosine_sample_residual.restype = ctypes.c_int

_lib.cosine_verify_tree.argtypes = [_P, _P, _i32, _i32, _i32, _i32, _P, _P, _P, _P, _i64, _f32, _P, _i64,
                                    _P, _P, _u32, ctypes.c_int, _P, _P, _P, _P]
_lib.cosine_verify_tree.restype = ctypes.c_int
_lib.cosine_verify_tree_lazy.argtypes = _lib.cosine_verify_tree.argtypes
_lib.cosine_fuse_step.argtypes = [_P, _P, _i32, _i32, _P, _i64, _f32, _P, _P, _P, _P, _P]
_lib.cosine_fuse_step.restype = ctypes.c_int
_lib.cosine_route_update.argtypes = [_P, _P, _i32, _i32, _i32, _P, _P, _P, _i64, _P, _P, _i64, _i64, ctypes.c_int,
                                     _P, _f32, _P, _P, _P]
_lib.cosine_route_update.restype = ctypes.c_int
_lib.cosine_tree_select.argtypes = [_P, _P, _i32, _i32, _i32, _P, _P, _i32, _P, _P, _P, _P, _P]
_lib.cosine_tree_select.restype = ctypes.c_int
_lib.cosine_verify_tree_lazy.restype = ctypes.c_int
_lib.cosine_verify_init_vgroup.argtypes = [ctypes.POINTER(cosine_config_t), _i32, ctypes.POINTER(_P)]
_lib.cosine_verify_init_vgroup.restype = ctypes.c_int
_lib.cosine_verify_batch_vgroup.argtypes = [ctypes.POINTER(_P), _i32, _P, _i32, _i32, _i32, ctypes.POINTER(_P), _i64,
                                            _f32, ctypes.POINTER(_P), _i64, _P, _P, _P, _u32, ctypes.c_int,
                                            ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P), _i32]
_lib.cosine_verify_batch_vgroup.restype = ctypes.c_int
_lib.cosine_nccl_unique_id.argtypes = [_P, _i64]
_lib.cosine_nccl_unique_id.restype = ctypes.c_int
_lib.cosine_profile_enable.argtypes = [_P, _i32]
_lib.cosine_profile_enable.restype = ctypes.c_int
_lib.cosine_profile_read.argtypes = [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i32)]
_lib.cosine_profile_read.restype = ctypes.c_int

EXPORTED_SYMBOLS = ("cosine_verify_init", "cosine_verify_destroy", "cosine_last_error",
                    "cosine_fuse_drafts", "cosine_verify_batch", "cosine_sample_residual",
                    "cosine_last_launch_count", "cosine_profile_enable", "cosine_profile_read",
                    "cosine_verify_tree", "cosine_nccl_unique_id", "cosine_verify_batch_lazy",
                    "cosine_verify_tree_lazy", "cosine_fuse_step",
                    "cosine_route_update", "cosine_tree_select", "cosine_verify_init_vgroup",
                    "cosine_verify_batch_vgroup", "cosine_exchange_mode")
NCCL_UNIQUE_ID_BYTES = 128


class CosineError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream, device):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _check(rc, ctx):
    if rc != 0:
        raise CosineError(rc, _lib.cosine_last_error(ctx).decode())


_DT = {torch.bfloat16: BF16, torch.float32: F32}


class Context:
    """Opaque cosine_ctx_t handle (passed straight to the C functions)."""

    def __init__(self, handle, cfg):
        self._as_parameter_ = handle
        self.cfg = cfg
        self.device = cfg.device
        self.vocab_size = cfg.vocab_size
        self.nranks, self.rank = cfg.nranks, cfg.rank
        self.vocab_begin, self.vocab_end = cfg.vocab_begin, cfg.vocab_end

    def __repr__(self):
        return (f"Context(V={self.vocab_size}, shard=[{self.vocab_begin}, {self.vocab_end}), "
                f"rank={self.rank}/{self.nranks}, device={self.device})")


def cosine_nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 calls this and broadcasts the bytes)."""
    buf = ctypes.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    _check(_lib.cosine_nccl_unique_id(buf, NCCL_UNIQUE_ID_BYTES), None)
    return buf.raw


def cosine_verify_init(vocab_size: int, *, device: int = 0, max_batch: int, max_draft_len: int,
                       max_drafters: int, target_dtype=torch.bfloat16, draft_dtype=torch.bfloat16,
                       draft_kind: int = DRAFT_PROBS, seed: int = 0, cluster_size: int = 0,
                       max_tree_nodes: int = 0, nranks: int = 1, rank: int = 0,
                       vocab_begin: int = 0, vocab_end: int | None = None,
                       nccl_unique_id: bytes | None = None, exchange: int = 0):
    """Create a context on `device`; returns a Context.  nranks > 1: vocabulary-sharded over
    nranks GPUs, this rank holding columns [vocab_begin, vocab_end) (collective init)."""
    vocab_end = vocab_size if vocab_end is None else vocab_end
    uid = None
    if nccl_unique_id is not None:
        uid = ctypes.create_string_buffer(bytes(nccl_unique_id), NCCL_UNIQUE_ID_BYTES)
    cfg = cosine_config_t(device=device, vocab_size=vocab_size, vocab_begin=vocab_begin,
                          vocab_end=vocab_end, max_batch=max_batch, max_draft_len=max_draft_len,
                          max_drafters=max_drafters, max_tree_nodes=max_tree_nodes,
                          target_dtype=_DT[target_dtype], draft_dtype=_DT[draft_dtype],
                          draft_kind=draft_kind, seed=seed, nranks=nranks, rank=rank,
                          nccl_unique_id=ctypes.cast(uid, _P) if uid is not None else None,
                          cluster_size=cluster_size, exchange=exchange)
    h = _P()
    _check(_lib.cosine_verify_init(ctypes.byref(cfg), ctypes.byref(h)), None)
    return Context(h, cfg)


def cosine_verify_init_vgroup(vocab_size: int, shards, *, device: int = 0, max_batch: int, max_draft_len: int,
                              max_drafters: int, target_dtype=torch.bfloat16, draft_dtype=torch.bfloat16,
                              draft_kind: int = DRAFT_PROBS, seed: int = 0, cluster_size: int = 0):
    """G contexts of a virtual vocabulary-sharded group on one device (test / diagnostic):
    shards = [(begin, end)] per rank, tiling [0, vocab_size) in rank order."""
    G = len(shards)
    cfgs = (cosine_config_t * G)()
    for g, (b, e) in enumerate(shards):
        cfgs[g] = cosine_config_t(device=device, vocab_size=vocab_size, vocab_begin=b, vocab_end=e,
                                  max_batch=max_batch, max_draft_len=max_draft_len, max_drafters=max_drafters,
                                  max_tree_nodes=0, target_dtype=_DT[target_dtype], draft_dtype=_DT[draft_dtype],
                                  draft_kind=draft_kind, seed=seed, nranks=G, rank=g, nccl_unique_id=None,
                                  cluster_size=cluster_size)
    hs = (_P * G)()
    _check(_lib.cosine_verify_init_vgroup(cfgs, G, hs), None)
    return [Context(_P(hs[g]), cfgs[g]) for g in range(G)]


def cosine_verify_batch_vgroup(ctxs, targets, drafts, draft_tokens, request_ids, accept_lens, out_tokens, statuses,
                               *, temperature=1.0, draft_len=None, step=0, weight_mode=W_CONF, stream=None,
                               peer_exchange=False):
    """The collective sharded call of a virtual group: targets[g] [B][k+1][ld_t] / drafts[g]
    [B][k][N][ld_q] are rank g's column shards; outputs per rank.  peer_exchange: the in-kernel
    peer-memory exchange of multi-GPU calls instead of copies between the phases."""
    G = len(ctxs)
    B, kp1, ld_t = targets[0].shape
    N, ld_q = drafts[0].shape[2], drafts[0].shape[3]
    arr = lambda ts: (_P * G)(*[t.data_ptr() for t in ts])
    hs = (_P * G)(*[c._as_parameter_ for c in ctxs])
    rc = _lib.cosine_verify_batch_vgroup(hs, G, _stream(stream, targets[0].device), B, kp1 - 1, N, arr(targets),
                                         ld_t, temperature, arr(drafts), ld_q, _ptr(draft_tokens), _ptr(draft_len),
                                         _ptr(request_ids), step, weight_mode, arr(accept_lens), arr(out_tokens),
                                         arr(statuses), 1 if peer_exchange else 0)
    _check(rc, ctxs[0])


def cosine_verify_destroy(ctx) -> None:
    _check(_lib.cosine_verify_destroy(ctx), None)


def cosine_last_launch_count(ctx) -> int:
    return int(_lib.cosine_last_launch_count(ctx))


EXCHANGE_MODES = {0: "none", 1: "nccl all-gathers", 2: "in-kernel nvlink peer writes", 3: "virtual group"}


def cosine_exchange_mode(ctx) -> str:
    return EXCHANGE_MODES.get(int(_lib.cosine_exchange_mode(ctx)), "?")


def cosine_profile_enable(ctx, enable: bool = True) -> None:
    _check(_lib.cosine_profile_enable(ctx, int(bool(enable))), ctx)


def cosine_profile_read(ctx):
    """-> (summed ms of the bracketed stats-kernel launches, number of launches)."""
    t = ctypes.c_double()
    n = _i32()
    _check(_lib.cosine_profile_read(ctx, ctypes.byref(t), ctypes.byref(n)), ctx)
    return t.value, n.value


def cosine_fuse_drafts(ctx, draft, draft_tokens, request_ids, fused_tokens, status, *, step=0,
                       temperature=1.0, weight_mode=W_CONF, select_mode=SEL_ARGMAX, weights=None,
                       draft_norm=None, fused_q=None, stream=None):
    B, k, N, ld_q = draft.shape
    ld_fq = fused_q.shape[-1] if fused_q is not None else 0
    rc = _lib.cosine_fuse_drafts(ctx, _stream(stream, draft.device), B, k, N, _ptr(draft), ld_q,
                                 _ptr(draft_tokens), _ptr(request_ids), step, temperature,
                                 weight_mode, select_mode, _ptr(fused_tokens), _ptr(weights),
                                 _ptr(draft_norm), _ptr(fused_q), ld_fq, _ptr(status))
    _check(rc, ctx)


def cosine_verify_batch(ctx, target_logits, draft, draft_tokens, request_ids, accept_len, out_tokens,
                        status, *, temperature=1.0, draft_len=None, step=0, weight_mode=W_CONF,
                        select_mode=SEL_ARGMAX, debug=None, stream=None):
    """target_logits [B][k+1][ld_t], draft [B][k][N][ld_q] (contiguous, on the ctx's device)."""
    B, kp1, ld_t = target_logits.shape
    N, ld_q = draft.shape[2], draft.shape[3]
    dbg = None
    if debug is not None:
        dbg = cosine_debug_t(**{f: _ptr(debug.get(f)) for f, _ in cosine_debug_t._fields_})
    rc = _lib.cosine_verify_batch(ctx, _stream(stream, target_logits.device), B, kp1 - 1, N,
                                  _ptr(target_logits), ld_t, temperature, _ptr(draft), ld_q,
                                  _ptr(draft_tokens), _ptr(draft_len), _ptr(request_ids), step,
                                  weight_mode, select_mode, _ptr(accept_len), _ptr(out_tokens),
                                  _ptr(status), ctypes.byref(dbg) if dbg is not None else None)
    _check(rc, ctx)


def cosine_verify_batch_lazy(ctx, target_logits, draft, draft_tokens, request_ids, accept_len, out_tokens,
                             status, *, temperature=1.0, draft_len=None, step=0, weight_mode=W_CONF,
                             debug=None, stream=None):
    """Early-exit verification (NEXT-1): same arguments / outputs as cosine_verify_batch."""
    B, kp1, ld_t = target_logits.shape
    N, ld_q = draft.shape[2], draft.shape[3]
    dbg = None
    if debug is not None:
        dbg = cosine_debug_t(**{f: _ptr(debug.get(f)) for f, _ in cosine_debug_t._fields_})
    rc = _lib.cosine_verify_batch_lazy(ctx, _stream(stream, target_logits.device), B, kp1 - 1, N,
                                       _ptr(target_logits), ld_t, temperature, _ptr(draft), ld_q,
                                       _ptr(draft_tokens), _ptr(draft_len), _ptr(request_ids), step,
                                       weight_mode, _ptr(accept_len), _ptr(out_tokens), _ptr(status),
                                       ctypes.byref(dbg) if dbg is not None else None)
    _check(rc, ctx)


def cosine_verify_tree(ctx, parent, node_token, internal_row, target, draft, node_draft_tokens,
                       request_ids, accept_len, accepted_nodes, out_tokens, status, *, temperature=1.0,
                       step=0, weight_mode=W_CONF, stream=None, lazy=False):
    """parent / node_token / internal_row [B][J+1], target [B][J+1][ld_t], draft [B][I][N][ld_q].
    lazy=True: cosine_verify_tree_lazy (path-only reads, NEXT-1)."""
    B, nn, ld_t = target.shape
    I, N, ld_q = draft.shape[1], draft.shape[2], draft.shape[3]
    fn = _lib.cosine_verify_tree_lazy if lazy else _lib.cosine_verify_tree
    rc = fn(ctx, _stream(stream, target.device), B, nn - 1, I, N, _ptr(parent),
                                 _ptr(node_token), _ptr(internal_row), _ptr(target), ld_t, temperature,
                                 _ptr(draft), ld_q, _ptr(node_draft_tokens), _ptr(request_ids), step,
                                 weight_mode, _ptr(accept_len), _ptr(accepted_nodes), _ptr(out_tokens),
                                 _ptr(status))
    _check(rc, ctx)


def cosine_sample_residual(ctx, target_rows, node_ids, request_ids, out_token, status, *,
                           temperature=1.0, row_max=None, row_sumexp=None, draft_rows=None,
                           weights=None, draft_norm=None, step=0, stream=None):
    B, ld_t = target_rows.shape
    N = draft_rows.shape[1] if draft_rows is not None else 0
    ld_q = draft_rows.shape[2] if draft_rows is not None else 0
    rc = _lib.cosine_sample_residual(ctx, _stream(stream, target_rows.device), B, _ptr(target_rows),
                                     ld_t, temperature, _ptr(row_max), _ptr(row_sumexp),
                                     _ptr(draft_rows), ld_q, _ptr(weights), _ptr(draft_norm), N,
                                     _ptr(node_ids), _ptr(request_ids), step, _ptr(out_token),
                                     _ptr(status))
    _check(rc, ctx)


def cosine_fuse_step(ctx, logits, own_tokens, conf, fused_token, winner, status, *, temperature=1.0,
                     stream=None):
    """Drafter-side Fuse of one iteration (NEXT-2): logits [B][N][ld] -> own_tokens [B][N],
    conf [B][N], fused_token [B], winner [B], status [B]."""
    B, N, ld = logits.shape
    rc = _lib.cosine_fuse_step(ctx, _stream(stream, logits.device), B, N, _ptr(logits), ld, temperature,
                               _ptr(own_tokens), _ptr(conf), _ptr(fused_token), _ptr(winner), _ptr(status))
    _check(rc, ctx)


def cosine_route_update(ctx, draft_tokens, conf, accepted, accept_len, emb, M, status, *, participating=None,
                        decay=0.9, d_out=None, stream=None):
    """Routing feedback (NEXT-3): draft_tokens / conf [B][N][K], accepted [B][>=K], accept_len [B],
    emb [V][H] (bf16 / fp32), M [B][N] fp32 updated in place, status [B]."""
    B, N, K = draft_tokens.shape
    H = emb.shape[1]
    rc = _lib.cosine_route_update(ctx, _stream(stream, M.device), B, N, K, _ptr(draft_tokens), _ptr(conf),
                                  _ptr(accepted), accepted.shape[1], _ptr(accept_len), _ptr(emb), H,
                                  emb.stride(0), _DT[emb.dtype], _ptr(participating), decay, _ptr(M),
                                  _ptr(d_out), _ptr(status))
    _check(rc, ctx)


def cosine_tree_select(ctx, tokens, conf, budget, n_nodes, parent, token, score, depth, *, stream=None):
    """TreeSelection (NEXT-4): tokens / conf [B][S][K] -> n_nodes [B], parent / token / score / depth
    [B][budget + 1] (breadth-first numbering, ready for cosine_verify_tree)."""
    B, S, K = tokens.shape
    rc = _lib.cosine_tree_select(ctx, _stream(stream, tokens.device), B, S, K, _ptr(tokens), _ptr(conf), budget,
                                 _ptr(n_nodes), _ptr(parent), _ptr(token), _ptr(score), _ptr(depth))
    _check(rc, ctx)
