"""ctypes marshalling for the fp64 C oracle (TEST INFRASTRUCTURE ONLY).

Argument marshalling only: every step of the method runs in ``cosine_oracle.c``.
All float inputs are converted to fp64 numpy arrays (exactly, from bf16 / fp32).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cosine_oracle.c")
_LIB_PATH = os.path.join(_HERE, "_build", "libcosine_oracle.so")

TAG_ACCEPT, TAG_SAMPLE, TAG_FUSE, TAG_TREE_GEN = 0, 1, 2, 3
W_CONF, W_WINNER, W_UNIFORM, W_POINT = 0, 1, 2, 3
SEL_ARGMAX, SEL_SAMPLE = 0, 1
DRAFT_PROBS, DRAFT_LOGITS = 0, 1
ST_OK, ST_ZERO_PROB, ST_TOKEN_RANGE, ST_NONFINITE, ST_EMPTY, ST_BAD_LEN, ST_BAD_TREE = range(7)
INFO_DEGENERATE = 0x100

__all__ = [
    "build", "lib", "philox4x32_10", "uniform", "invcdf", "softmax", "residual",
    "verify_batch", "verify_batch_parallel", "by_request", "fuse_drafts", "sample_residual", "verify_tree", "fuse_step", "route_update", "tree_select",
    "TAG_ACCEPT", "TAG_SAMPLE", "TAG_FUSE", "TAG_TREE_GEN",
    "W_CONF", "W_WINNER", "W_UNIFORM", "W_POINT", "SEL_ARGMAX", "SEL_SAMPLE",
    "DRAFT_PROBS", "DRAFT_LOGITS", "ST_OK", "ST_ZERO_PROB", "ST_TOKEN_RANGE",
    "ST_NONFINITE", "ST_EMPTY", "ST_BAD_LEN", "ST_BAD_TREE", "INFO_DEGENERATE",
]


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no fast-math, no FMA contraction)."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "cosine_oracle.h"))
    ):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-Wall", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None

_P = ctypes.c_void_p
_i32, _i64, _u32, _u64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.orc_philox4x32_10.argtypes = [_P, _P, _P]
        L.orc_uniform.argtypes = [_u64, _u64, _u32, _u32, _u32]
        L.orc_uniform.restype = _f64
        L.orc_invcdf.argtypes = [_P, _i64, _f64, _P]
        L.orc_invcdf.restype = _i64
        L.orc_softmax.argtypes = [_P, _i64, _f64, _P, _P, _P]
        L.orc_residual.argtypes = [_P, _P, _i64, _P]
        L.orc_verify_batch.argtypes = ([_i32, _i32, _i32, _i64, _P, _f64, _P, _i32, _P, _P, _P, _u64,
                                        _u32, _i32, _i32, _P, _P, _P] + [_P] * 11)
        L.orc_fuse_drafts.argtypes = [_i32, _i32, _i32, _i64, _P, _i32, _f64, _P, _P, _u64, _u32,
                                      _i32, _i32, _P, _P, _P, _P, _P, _P]
        L.orc_sample_residual.argtypes = [_i32, _i64, _P, _f64, _P, _P, _P, _i32, _P, _P, _P, _P,
                                          _u64, _u32, _P, _P, _P, _P]
        L.orc_verify_tree.argtypes = [_i32, _i32, _i32, _i32, _i64, _P, _P, _P, _P, _f64, _P, _i32,
                                      _P, _P, _u64, _u32, _i32, _P, _P, _P, _P, _P]
        L.orc_fuse_step.argtypes = [_i32, _i32, _i64, _P, _f64, _P, _P, _P, _P, _P, _P]
        L.orc_tree_select.argtypes = [_i32, _i32, _i32, _P, _P, _i32, _P, _P, _P, _P, _P]
        L.orc_route_update.argtypes = [_i32, _i32, _i32, _i64, _i64, _P, _P, _P, _i64, _P, _P, _P, _f64, _f64,
                                       _P, _P, _P]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64arr(x):
    if x is None:
        return None
    if hasattr(x, "detach"):  # torch tensor (bf16 / fp32) -> exact fp64
        x = x.detach().to("cpu").double().numpy()
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _arr(x, dt):
    if x is None:
        return None
    if hasattr(x, "detach"):
        x = x.detach().to("cpu").numpy()
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def uniform(seed, request_id, node, step, tag):
    return lib().orc_uniform(int(seed), int(request_id), int(node), int(step), int(tag))


def invcdf(w, u, with_margin=False):
    w = _f64arr(w)
    m = np.zeros(1)
    y = lib().orc_invcdf(_ptr(w), w.size, float(u), _ptr(m))
    return (int(y), float(m[0])) if with_margin else int(y)


def softmax(l, T):
    l = _f64arr(l)
    p = np.zeros_like(l)
    M = np.zeros(1)
    S = np.zeros(1)
    st = lib().orc_softmax(_ptr(l), l.size, float(T), _ptr(p), _ptr(M), _ptr(S))
    return st, p, float(M[0]), float(S[0])


def residual(o, q):
    o, q = _f64arr(o), _f64arr(q)
    r = np.zeros_like(o)
    deg = lib().orc_residual(_ptr(o), _ptr(q), o.size, _ptr(r))
    return bool(deg), r


def verify_batch(target, draft, draft_tokens, request_ids, *, temperature=1.0, seed=0, step=0,
                 draft_len=None, draft_kind=DRAFT_PROBS, weight_mode=W_CONF, select_mode=SEL_ARGMAX,
                 vocab=None):
    """target [B][k+1][V] logits, draft [B][k][N][V]; returns a dict of numpy arrays."""
    t = _f64arr(target)
    d = _f64arr(draft)
    B, kp1, V = t.shape
    k = kp1 - 1
    N = d.shape[2]
    if vocab is not None:  # columns beyond the vocabulary (row padding) are dropped
        t, d, V = np.ascontiguousarray(t[..., :vocab]), np.ascontiguousarray(d[..., :vocab]), vocab
    X = _arr(draft_tokens, np.int32)
    rid = _arr(request_ids, np.uint64)
    dl = _arr(draft_len, np.int32)
    out = dict(
        accept_len=np.zeros(B, np.int32), out_tokens=np.zeros((B, k + 1), np.int32),
        status=np.zeros(B, np.int32), p_x=np.full((B, k), np.nan), q_x=np.full((B, k), np.nan),
        M=np.full((B, k + 1), np.nan), S=np.full((B, k + 1), np.nan),
        sigma=np.full((B, k, N), np.nan), conf=np.full((B, k, N), np.nan),
        weights=np.full((B, k, N), np.nan), fused_tokens=np.full((B, k), -1, np.int32),
        u=np.full((B, k), np.nan), Z=np.full(B, np.nan), tie_margin=np.full(B, np.inf),
    )
    rc = lib().orc_verify_batch(
        B, k, N, V, _ptr(t), float(temperature), _ptr(d), int(draft_kind), _ptr(X), _ptr(dl),
        _ptr(rid), int(seed), int(step), int(weight_mode), int(select_mode),
        _ptr(out["accept_len"]), _ptr(out["out_tokens"]), _ptr(out["status"]),
        _ptr(out["p_x"]), _ptr(out["q_x"]), _ptr(out["M"]), _ptr(out["S"]), _ptr(out["sigma"]),
        _ptr(out["conf"]), _ptr(out["weights"]), _ptr(out["fused_tokens"]), _ptr(out["u"]),
        _ptr(out["Z"]), _ptr(out["tie_margin"]))
    if rc != 0:
        raise ValueError("oracle verify_batch: invalid argument")
    return out


def by_request(fn, *batch_args, threads=None, **kw):
    """fn(*slices, **kw) over single-request slices of the batch-major arguments (None stays
    None) on `threads` host threads (default: all cores); the per-request result dicts are
    concatenated.  Requests are independent (Alg. 2 "foreach draft ... in parallel") and
    every random draw is keyed by the global request id (reading #8), so the result equals the
    whole-batch call; ctypes releases the GIL inside the C oracle, so requests run concurrently
    and only `threads` requests are converted to fp64 at a time."""
    from concurrent.futures import ThreadPoolExecutor
    B = int(batch_args[0].shape[0])
    threads = max(1, min(B, threads or os.cpu_count() or 1))

    def one(b):
        return fn(*[None if a is None else a[b:b + 1] for a in batch_args], **kw)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        parts = list(ex.map(one, range(B)))
    return {n: np.concatenate([r[n] for r in parts]) for n in parts[0]}


def verify_batch_parallel(target, draft, draft_tokens, request_ids, *, threads=None, draft_len=None,
                          **kw):
    """verify_batch, one request per task on `threads` host threads (by_request)."""
    def fn(t, d, x, r, dl):
        return verify_batch(t, d, x, r, draft_len=dl, **kw)
    return by_request(fn, target, draft, draft_tokens, request_ids, draft_len, threads=threads)


def fuse_drafts(draft, draft_tokens, request_ids, *, temperature=1.0, seed=0, step=0,
                draft_kind=DRAFT_PROBS, weight_mode=W_CONF, select_mode=SEL_ARGMAX, want_q=False,
                vocab=None):
    d = _f64arr(draft)
    B, k, N, V = d.shape
    if vocab is not None:
        d, V = np.ascontiguousarray(d[..., :vocab]), vocab
    X = _arr(draft_tokens, np.int32)
    rid = _arr(request_ids, np.uint64)
    out = dict(fused_tokens=np.zeros((B, k), np.int32), weights=np.full((B, k, N), np.nan),
               draft_norm=np.full((B, k, N), np.nan), status=np.zeros(B, np.int32),
               tie_margin=np.full(B, np.inf),
               fused_q=np.full((B, k, V), np.nan) if want_q else None)
    rc = lib().orc_fuse_drafts(B, k, N, V, _ptr(d), int(draft_kind), float(temperature), _ptr(X),
                               _ptr(rid), int(seed), int(step), int(weight_mode), int(select_mode),
                               _ptr(out["fused_tokens"]), _ptr(out["weights"]), _ptr(out["draft_norm"]),
                               _ptr(out["fused_q"]), _ptr(out["status"]), _ptr(out["tie_margin"]))
    if rc != 0:
        raise ValueError("oracle fuse_drafts: invalid argument")
    return out


def sample_residual(target, node_ids, request_ids, *, temperature=1.0, seed=0, step=0,
                    row_max=None, row_sumexp=None, draft=None, weights=None, draft_norm=None,
                    vocab=None):
    t = _f64arr(target)
    B, V = t.shape
    d = _f64arr(draft)
    if vocab is not None:
        t = np.ascontiguousarray(t[:, :vocab])
        d = None if d is None else np.ascontiguousarray(d[..., :vocab])
        V = vocab
    N = 0 if d is None else d.shape[1]
    w = _f64arr(weights)
    s = _f64arr(draft_norm)
    rm, rs = _f64arr(row_max), _f64arr(row_sumexp)
    nid = _arr(node_ids, np.uint32)
    rid = _arr(request_ids, np.uint64)
    out = dict(out_token=np.zeros(B, np.int32), status=np.zeros(B, np.int32),
               Z=np.full(B, np.nan), tie_margin=np.full(B, np.inf))
    rc = lib().orc_sample_residual(B, V, _ptr(t), float(temperature), _ptr(rm), _ptr(rs), _ptr(d),
                                   N, _ptr(w), _ptr(s), _ptr(nid), _ptr(rid), int(seed), int(step),
                                   _ptr(out["out_token"]), _ptr(out["status"]), _ptr(out["Z"]),
                                   _ptr(out["tie_margin"]))
    if rc != 0:
        raise ValueError("oracle sample_residual: invalid argument")
    return out


def verify_tree(parent, node_token, internal_row, target, draft, node_draft_tokens, request_ids, *,
                temperature=1.0, seed=0, step=0, draft_kind=DRAFT_PROBS, weight_mode=W_CONF,
                vocab=None):
    par = _arr(parent, np.int32)
    tok = _arr(node_token, np.int32)
    irow = _arr(internal_row, np.int32)
    t = _f64arr(target)
    d = _f64arr(draft)
    B, nn, V = t.shape
    I, N = d.shape[1], d.shape[2]
    if vocab is not None:
        t, d, V = np.ascontiguousarray(t[..., :vocab]), np.ascontiguousarray(d[..., :vocab]), vocab
    X = _arr(node_draft_tokens, np.int32)
    rid = _arr(request_ids, np.uint64)
    out = dict(accept_len=np.zeros(B, np.int32), accepted_nodes=np.zeros((B, nn), np.int32),
               out_tokens=np.zeros((B, nn), np.int32), status=np.zeros(B, np.int32),
               tie_margin=np.full(B, np.inf))
    rc = lib().orc_verify_tree(B, nn - 1, I, N, V, _ptr(par), _ptr(tok), _ptr(irow), _ptr(t),
                               float(temperature), _ptr(d), int(draft_kind), _ptr(X), _ptr(rid),
                               int(seed), int(step), int(weight_mode), _ptr(out["accept_len"]),
                               _ptr(out["accepted_nodes"]), _ptr(out["out_tokens"]),
                               _ptr(out["status"]), _ptr(out["tie_margin"]))
    if rc != 0:
        raise ValueError("oracle verify_tree: invalid argument")
    return out


def fuse_step(logits, *, temperature=1.0, vocab=None):
    """Drafter-side Fuse of one iteration (NEXT-2): logits [B][N][V] -> dict(own_tokens, conf,
    fused_token, winner, status, conf_gap)."""
    l = _f64arr(logits)
    if vocab is not None:
        l = np.ascontiguousarray(l[..., :vocab])
    B, N, V = l.shape
    out = dict(own_tokens=np.zeros((B, N), np.int32), conf=np.zeros((B, N)), fused_token=np.zeros(B, np.int32),
               winner=np.zeros(B, np.int32), status=np.zeros(B, np.int32), conf_gap=np.zeros(B))
    rc = lib().orc_fuse_step(B, N, V, _ptr(l), float(temperature), _ptr(out["own_tokens"]), _ptr(out["conf"]),
                             _ptr(out["fused_token"]), _ptr(out["winner"]), _ptr(out["status"]),
                             _ptr(out["conf_gap"]))
    if rc != 0:
        raise ValueError("oracle fuse_step: invalid argument")
    return out


def route_update(draft_tokens, conf, accepted, accept_len, emb, M, *, participating=None, decay=0.9,
                 eps=1e-6):
    """Routing feedback (NEXT-3, Eqs. 1-2): returns dict(M (updated copy), d, status)."""
    X = _arr(draft_tokens, np.int32)
    B, N, K = X.shape
    c = _f64arr(conf)
    acc = _arr(accepted, np.int32)
    L = _arr(accept_len, np.int32)
    E = _f64arr(emb)
    V, Hd = E.shape
    Mo = _f64arr(M).copy()
    part = None if participating is None else _arr(participating, np.uint8)
    d = np.zeros((B, N, K))
    st = np.zeros(B, np.int32)
    rc = lib().orc_route_update(B, N, K, V, Hd, _ptr(X), _ptr(c), _ptr(acc), acc.shape[1], _ptr(L), _ptr(E),
                                _ptr(part), float(decay), float(eps), _ptr(Mo), _ptr(d), _ptr(st))
    if rc != 0:
        raise ValueError("oracle route_update: invalid argument")
    return dict(M=Mo, d=d, status=st)


def tree_select(tokens, conf, budget):
    """TreeSelection (NEXT-4): tokens / conf [B][S][K] -> dict(n_nodes, parent, token, score, depth)."""
    X = _arr(tokens, np.int32)
    C = _f64arr(conf)
    B, S, K = X.shape
    out = dict(n_nodes=np.zeros(B, np.int32), parent=np.zeros((B, budget + 1), np.int32),
               token=np.zeros((B, budget + 1), np.int32), score=np.zeros((B, budget + 1)),
               depth=np.zeros((B, budget + 1), np.int32))
    rc = lib().orc_tree_select(B, S, K, _ptr(X), _ptr(C), int(budget), _ptr(out["n_nodes"]), _ptr(out["parent"]),
                               _ptr(out["token"]), _ptr(out["score"]), _ptr(out["depth"]))
    if rc != 0:
        raise ValueError("oracle tree_select: invalid argument")
    return out
