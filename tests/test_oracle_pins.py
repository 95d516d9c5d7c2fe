"""Pins of the fp64 CPU oracle against what the paper and the mathematics fix (no GPU).

Every test cites the passage it checks.  A plausible mistake anywhere in the oracle
(a dropped term, a wrong sign or index, a transposed operand, a wrong Philox
constant or counter layout) fails at least one of them:

* Philox / uniforms  — Random123 known-answer vectors (golden file), uniformity.
* softmax            — scipy.special.softmax (library routine), masking / errors.
* inverse CDF        — numpy.searchsorted over numpy.cumsum (library routine).
* residual           — SPEC worked values S:72-74 and the invariant S:77.
* fusion (Eq. 4)     — S:291-293 examples and the tie rule.
* acceptance         — draft == target gives 100% acceptance; the closed form
                       P(accept) = sum_v min(p, q) by Monte Carlo.
* whole step         — exact rational enumeration (oracle/enum_check.py): the method
                       emits the target conditional at every position (P:126-127,
                       P:130-133); the oracle's realisations follow that exact law
                       (chi-square) in every mode, including the biased paper-literal
                       ARGMAX+CONF mode (reading #3).
* greedy             — T = 0 equals the argmax decode (numpy.argmax).
* tree               — a chain tree is bit-identical to the linear path;
                       the tree walk realises the enumerated law, which equals o.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.special
import scipy.stats

import oracle
from oracle import enum_check as ec

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------- Philox
def test_philox_known_answer_vectors():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt"))
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = oracle.philox4x32_10(v[0:4], v[4:6])
        assert [int(x) for x in out] == v[6:10]


def test_uniform_counter_layout_and_range():
    # U = (x0 >> 8) * 2^-24 of ctr = {rid_lo, rid_hi, node, (step << 4) | tag}, key = seed
    seed, rid, node, step, tag = 0x0123456789ABCDEF, 0xFEDCBA9876543210, 7, 3, 1
    x = oracle.philox4x32_10([rid & 0xffffffff, rid >> 32, node, (step << 4) | tag],
                             [seed & 0xffffffff, seed >> 32])
    assert oracle.uniform(seed, rid, node, step, tag) == (int(x[0]) >> 8) / 2 ** 24
    us = np.array([oracle.uniform(5, r, 1, 0, 0) for r in range(20000)])
    assert us.min() >= 0.0 and us.max() <= 1.0 - 2 ** -24
    counts, _ = np.histogram(us, bins=20, range=(0, 1))
    assert scipy.stats.chisquare(counts).pvalue > 1e-4
    # distinct tags / nodes / steps give independent streams
    a = np.array([oracle.uniform(5, r, 1, 0, 0) for r in range(2000)])
    b = np.array([oracle.uniform(5, r, 1, 0, 1) for r in range(2000)])
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.1


# --------------------------------------------------------------------------- softmax
@pytest.mark.parametrize("T", [1.0, 0.5, 2.0])
def test_softmax_matches_scipy(T):
    rng = np.random.default_rng(1)
    l = rng.normal(size=1000) * 5
    st, p, M, S = oracle.softmax(l, T)
    assert st == 0
    ref = scipy.special.softmax(l / T)
    np.testing.assert_allclose(p, ref, rtol=1e-12, atol=1e-300)
    assert M == pytest.approx((l / T).max(), rel=0, abs=0)
    assert S == pytest.approx(np.exp(l / T - M).sum(), rel=1e-13)


def test_softmax_masking_and_errors():
    st, p, _, _ = oracle.softmax([0.0, -np.inf, 0.0], 1.0)
    assert st == 0 and p.tolist() == [0.5, 0.0, 0.5]
    assert oracle.softmax([0.0, np.nan], 1.0)[0] == oracle.ST_NONFINITE
    assert oracle.softmax([0.0, np.inf], 1.0)[0] == oracle.ST_NONFINITE
    assert oracle.softmax([-np.inf, -np.inf], 1.0)[0] == oracle.ST_EMPTY


# --------------------------------------------------------------------------- inverse CDF
def test_invcdf_matches_searchsorted():
    rng = np.random.default_rng(2)
    for _ in range(300):
        V = int(rng.integers(1, 40))
        w = rng.random(V) * (rng.random(V) < 0.7)
        if w.sum() == 0:
            w[int(rng.integers(0, V))] = 1.0
        u = float(rng.random())
        c = np.cumsum(w)
        ref = int(np.searchsorted(c, u * c[-1], side="right"))  # smallest v with C(v) > t
        assert oracle.invcdf(w, u) == ref
    assert oracle.invcdf([0.0, 0.0], 0.3) == -1
    assert oracle.invcdf([0.0, 1.0, 0.0], 0.0) == 1  # zero-weight bins are never drawn


# --------------------------------------------------------------------------- residual
def test_residual_spec_examples():
    g = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))
    for ex in g["residual"]:
        deg, r = oracle.residual(ex["o"], ex["q"])
        if ex.get("degenerate"):
            assert deg
        else:
            assert not deg
            np.testing.assert_allclose(r, ex["r"], atol=1e-15)


def test_residual_invariant():
    # sums to 1 when non-degenerate and is 0 wherever q >= o
    rng = np.random.default_rng(3)
    for _ in range(200):
        V = int(rng.integers(2, 30))
        o, q = rng.random(V), rng.random(V)
        o, q = o / o.sum(), q / q.sum()
        deg, r = oracle.residual(o, q)
        assert not deg
        assert abs(r.sum() - 1) < 1e-12
        assert np.all(r[q >= o] == 0) and np.all(r[q < o] > 0)


# --------------------------------------------------------------------------- fusion
def _rows_with_conf(conf, V=2):
    """Drafter n's row puts probability conf[n] on token 0 (its own token) and the rest on 1."""
    N = len(conf)
    d = np.zeros((1, 1, N, V))
    for n, c in enumerate(conf):
        d[0, 0, n, 0] = c
        d[0, 0, n, 1] = 1 - c
    return d


def test_fusion_spec_examples():
    g = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))
    for ex in g["fuse"]:
        conf = ex["conf"]
        N = len(conf)
        d = _rows_with_conf(conf, V=2 + N)
        # each drafter's own token: 0 for all, but make them distinguishable by moving drafter n's
        # confident mass to token n (same confidence, distinct tokens)
        d2 = np.zeros_like(d)
        for n in range(N):
            d2[0, 0, n, n] = d[0, 0, n, 0]
            d2[0, 0, n, N] = d[0, 0, n, 1]
        X = np.arange(N, dtype=np.int32).reshape(1, 1, N)
        for wm in (oracle.W_CONF, oracle.W_WINNER, oracle.W_UNIFORM, oracle.W_POINT):
            r = oracle.fuse_drafts(d2, X, [0], weight_mode=wm)
            assert r["status"][0] == 0
            assert r["fused_tokens"][0, 0] == ex["expect_node"]  # Eq. 4 argmax, ties -> lowest n
        r = oracle.fuse_drafts(d2, X, [0], weight_mode=oracle.W_CONF, want_q=True)
        c = np.array(conf)
        np.testing.assert_allclose(r["weights"][0, 0], c / c.sum(), rtol=1e-14)
        np.testing.assert_allclose(r["draft_norm"][0, 0], np.ones(N), rtol=1e-14)
        # fused q = sum_n w_n q_n (reading #2)
        np.testing.assert_allclose(r["fused_q"][0, 0], (c / c.sum()) @ d2[0, 0], rtol=1e-13)


def test_fusion_renormalises_bf16_rows():
    # reading #6: a drafter row that does not sum to 1 is renormalised by its sum
    d = np.array([[[[0.2, 0.2, 0.1]]]])  # sums to 0.5
    r = oracle.fuse_drafts(d, np.array([[[1]]], np.int32), [0], want_q=True)
    assert r["draft_norm"][0, 0, 0] == pytest.approx(0.5)
    np.testing.assert_allclose(r["fused_q"][0, 0], [0.4, 0.4, 0.2], rtol=1e-14)


# --------------------------------------------------------------------------- acceptance pins
def test_draft_equals_target_accepts_everything():
    # q = o  =>  min(1, o/q) = 1; with identical logits rows (N = 1, LOGITS)
    rng = np.random.default_rng(4)
    B, k, V = 64, 6, 300
    t = rng.normal(size=(B, k + 1, V)) * 5
    d = t[:, :k, None, :].copy()
    X = np.zeros((B, k, 1), np.int32)
    for b in range(B):
        for i in range(k):
            p = scipy.special.softmax(t[b, i])
            X[b, i, 0] = rng.choice(V, p=p)
    for T in (1.0, 0.7):
        r = oracle.verify_batch(t, d, X, np.arange(B), temperature=T, draft_kind=oracle.DRAFT_LOGITS)
        assert (r["status"] == 0).all()
        assert (r["accept_len"] == k).all()
        np.testing.assert_array_equal(r["out_tokens"][:, :k], X[:, :, 0])


def _mc_bound(p, n):
    return 4.5 * math.sqrt(p * (1 - p) / n) + 1e-9


@pytest.mark.parametrize("N,wm", [(1, oracle.W_CONF), (3, oracle.W_UNIFORM)])
def test_closed_form_acceptance_rate(N, wm):
    # x ~ q (SAMPLE) accepted w.p. min(1, p/q)  =>  P(accept) = sum_v min(p(v), q(v))
    rng = np.random.default_rng(5 + N)
    V, n = 12, 40000
    l = rng.normal(size=V) * 1.5
    p = scipy.special.softmax(l)
    qs = rng.dirichlet(np.ones(V), size=N)
    q = qs.mean(0)
    t = np.broadcast_to(np.stack([l, l]), (n, 2, V)).copy()
    d = np.broadcast_to(qs[None, None], (n, 1, N, V)).copy()
    X = np.zeros((n, 1, N), np.int32)  # own tokens only enter the (unused) CONF weights
    for m in range(N):
        X[:, 0, m] = int(np.argmax(qs[m]))
    r = oracle.verify_batch(t, d, X, np.arange(n), seed=11, weight_mode=wm,
                            select_mode=oracle.SEL_SAMPLE)
    rate = (r["accept_len"] >= 1).mean()
    expect = np.minimum(p, q).sum()
    assert abs(rate - expect) < _mc_bound(expect, n)


def test_ab_example():
    # o = (.5, .5), q = (1, 0), draft a: accept w.p. 0.5; the emitted token is o-distributed
    g = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))["ab_example"]
    n = 40000
    t = np.log(np.broadcast_to(np.array(g["o"]), (n, 2, 2)))
    d = np.broadcast_to(np.array(g["q"]), (n, 1, 1, 2)).copy()
    X = np.zeros((n, 1, 1), np.int32)
    r = oracle.verify_batch(t, d, X, np.arange(n), seed=3)
    acc = (r["accept_len"] == 1).mean()
    assert abs(acc - g["accept_prob"]) < _mc_bound(0.5, n)
    first = r["out_tokens"][:, 0]
    assert abs((first == 0).mean() - g["marginal"][0]) < _mc_bound(0.5, n)
    assert (first[r["accept_len"] == 0] == 1).all()  # residual of (.5,.5)-(1,0) is (0,1)


# --------------------------------------------------------------------------- greedy
def test_greedy_is_argmax_decode():
    rng = np.random.default_rng(6)
    B, k, N, V = 50, 5, 3, 40
    t = np.round(rng.normal(size=(B, k + 1, V)) * 2)  # many exact ties: lowest index wins
    d = rng.dirichlet(np.ones(V), size=(B, k, N))
    X = rng.integers(0, V, (B, k, N)).astype(np.int32)
    # make every drafter token carry some mass
    for b in range(B):
        for i in range(k):
            for n in range(N):
                d[b, i, n, X[b, i, n]] += 0.1
    r = oracle.verify_batch(t, d, X, np.arange(B), temperature=0.0)
    am = np.argmax(t, axis=-1)
    for b in range(B):
        xs = r["fused_tokens"][b]
        L = next((i for i in range(k) if xs[i] != am[b, i]), k)
        assert r["accept_len"][b] == L
        assert list(r["out_tokens"][b, :L]) == list(xs[:L])
        assert r["out_tokens"][b, L] == am[b, L]


# --------------------------------------------------------------------------- exact enumeration
def _models(seed, V, depth, context_free=False):
    rng = np.random.default_rng(seed)
    if context_free:
        tabs = [ec.random_dist(rng, V) for _ in range(depth + 2)]
        return lambda prefix: tabs[len(prefix)]
    return ec.random_tabular_model(rng, V, depth)


EXACT_MODES = [(ec.W_CONF, ec.SEL_SAMPLE), (ec.W_WINNER, ec.SEL_SAMPLE),
               (ec.W_UNIFORM, ec.SEL_SAMPLE), (ec.W_POINT, ec.SEL_ARGMAX)]


@pytest.mark.parametrize("wm,sm", EXACT_MODES)
def test_enumeration_method_preserves_target(wm, sm):
    # P:126-127 / P:130-133: every emitted token ~ o(. | prefix), exactly
    for seed in range(6):
        V, gamma = 3, 2
        target = _models(100 + seed, V, gamma + 1)
        drafters = [_models(200 + seed * 7 + n, V, gamma + 1) for n in range(2)]
        law = ec.linear_law(target, drafters, gamma, wm, sm)
        assert sum(law.values()) == 1
        assert ec.max_tvd_to_target(law, target, V, gamma + 1) == 0


def test_enumeration_argmax_conf_is_biased():
    # reading #3: the paper-literal Eq. 4 argmax with a mixture q is not distribution exact
    worst = Fraction(0)
    for seed in range(10):
        V = 4
        target = _models(300 + seed, V, 2)
        drafters = [_models(400 + seed * 7 + n, V, 2) for n in range(2)]
        law = ec.linear_law(target, drafters, 1, ec.W_CONF, ec.SEL_ARGMAX)
        worst = max(worst, ec.max_tvd_to_target(law, target, V, 1))
    assert worst > Fraction(1, 100)


def _sample_linear_case(rng, target, drafters, k, n_req, V, wm):
    """Inputs along the fused path: X_n ~ q_n(. | prefix) and (ARGMAX) x* = Eq. 4's argmax."""
    N = len(drafters)
    t = np.zeros((n_req, k + 1, V))
    d = np.zeros((n_req, k, N, V))
    X = np.zeros((n_req, k, N), np.int32)
    for b in range(n_req):
        prefix = ()
        for i in range(k):
            t[b, i] = np.log(np.array([float(x) for x in target(prefix)]) + 1e-300)
            qs = [np.array([float(x) for x in dm(prefix)]) for dm in drafters]
            for n in range(N):
                d[b, i, n] = qs[n]
                X[b, i, n] = rng.choice(V, p=qs[n] / qs[n].sum())
            c = [qs[n][X[b, i, n]] for n in range(N)]
            nstar = int(np.argmax(c))
            prefix = prefix + (int(X[b, i, nstar]),)
        t[b, k] = np.log(np.array([float(x) for x in target(prefix)]) + 1e-300)
    return t, d, X


def _chi2_law(counts, law, n):
    keys = sorted(law)
    exp = np.array([float(law[k2]) * n for k2 in keys])
    obs = np.array([counts.get(k2, 0) for k2 in keys], dtype=float)
    assert sum(counts.get(k2, 0) for k2 in keys) == sum(counts.values()), "impossible outcome"
    small = exp < 5
    if small.any():
        exp = np.append(exp[~small], exp[small].sum())
        obs = np.append(obs[~small], obs[small].sum())
    return scipy.stats.chisquare(obs, exp).pvalue


@pytest.mark.parametrize("wm,sm,ctx_free", [
    (ec.W_CONF, ec.SEL_ARGMAX, False),   # paper-literal (biased) mode
    (ec.W_POINT, ec.SEL_ARGMAX, False),
    (ec.W_CONF, ec.SEL_SAMPLE, True),
    (ec.W_UNIFORM, ec.SEL_SAMPLE, True),
])
def test_oracle_realises_enumerated_law(wm, sm, ctx_free):
    V, k, n = 3, 2, 30000
    target = _models(500, V, k + 1, ctx_free)
    drafters = [_models(600 + j, V, k + 1, ctx_free) for j in range(2)]
    law = ec.linear_law(target, drafters, k, wm, sm)
    rng = np.random.default_rng(7)
    t, d, X = _sample_linear_case(rng, target, drafters, k, n, V, wm)
    r = oracle.verify_batch(t, d, X, np.arange(n), seed=123, weight_mode=wm, select_mode=sm)
    assert (r["status"] == 0).all()
    counts = {}
    for b in range(n):
        seq = tuple(int(x) for x in r["out_tokens"][b, : r["accept_len"][b] + 1])
        counts[seq] = counts.get(seq, 0) + 1
    assert _chi2_law(counts, law, n) > 1e-4


# --------------------------------------------------------------------------- errors
def test_error_statuses_and_isolation():
    rng = np.random.default_rng(8)
    B, k, N, V = 7, 3, 2, 20
    t = rng.normal(size=(B, k + 1, V))
    d = rng.dirichlet(np.ones(V), size=(B, k, N))
    X = rng.integers(0, V, (B, k, N)).astype(np.int32)
    dl = np.full(B, k, np.int32)
    d[1, 0, 1, X[1, 0, 1]] = 0.0                 # zero-probability own token
    X[2, 1, 0] = V                               # token out of range
    t[3, 2, 5] = np.nan                          # non-finite logit
    d[4, 1, 0, 3] = -0.1                         # negative probability
    t[5, 0, :] = -np.inf                         # empty row
    dl[6] = 0                                    # bad gamma
    r = oracle.verify_batch(t, d, X, np.arange(B), draft_len=dl)
    assert list(r["status"]) == [0, oracle.ST_ZERO_PROB, oracle.ST_TOKEN_RANGE, oracle.ST_NONFINITE,
                                 oracle.ST_NONFINITE, oracle.ST_EMPTY, oracle.ST_BAD_LEN]
    assert r["accept_len"][0] >= 0 and (r["accept_len"][1:] == -1).all()
    assert (r["out_tokens"][1:] == -1).all()


def test_rows_past_draft_len_are_ignored():
    rng = np.random.default_rng(9)
    B, k, N, V = 4, 4, 2, 30
    t = rng.normal(size=(B, k + 1, V))
    d = rng.dirichlet(np.ones(V), size=(B, k, N))
    X = rng.integers(0, V, (B, k, N)).astype(np.int32)
    dl = np.array([1, 2, 3, 4], np.int32)
    r1 = oracle.verify_batch(t, d, X, np.arange(B), draft_len=dl, seed=4)
    for b in range(B):
        t[b, dl[b] + 1:] = np.nan
        d[b, dl[b]:] = np.nan
    r2 = oracle.verify_batch(t, d, X, np.arange(B), draft_len=dl, seed=4)
    np.testing.assert_array_equal(r1["out_tokens"], r2["out_tokens"])
    assert (r2["status"] == 0).all() and (r2["accept_len"] <= dl).all()


def test_result_independent_of_batch_order():
    # reading #8: Philox keyed by global request id
    rng = np.random.default_rng(10)
    B, k, N, V = 6, 3, 2, 25
    t = rng.normal(size=(B, k + 1, V)) * 3
    d = rng.dirichlet(np.ones(V), size=(B, k, N))
    X = rng.integers(0, V, (B, k, N)).astype(np.int32)
    rid = np.arange(100, 100 + B)
    r1 = oracle.verify_batch(t, d, X, rid, seed=9)
    perm = rng.permutation(B)
    r2 = oracle.verify_batch(t[perm], d[perm], X[perm], rid[perm], seed=9)
    np.testing.assert_array_equal(r1["out_tokens"][perm], r2["out_tokens"])


# --------------------------------------------------------------------------- sample_residual
def test_sample_residual_matches_verify_path():
    rng = np.random.default_rng(12)
    B, k, N, V = 40, 3, 2, 60
    t = rng.normal(size=(B, k + 1, V)) * 3
    d = rng.dirichlet(np.ones(V) * 0.5, size=(B, k, N))
    X = np.zeros((B, k, N), np.int32)
    for b in range(B):
        for i in range(k):
            for n in range(N):
                X[b, i, n] = rng.choice(V, p=d[b, i, n])
    r = oracle.verify_batch(t, d, X, np.arange(B), seed=5)
    L = r["accept_len"]
    rows = t[np.arange(B), L]
    has_rej = L < k
    Lc = np.minimum(L, k - 1)
    s = oracle.sample_residual(rows[has_rej], L[has_rej].astype(np.uint32), np.arange(B)[has_rej],
                               seed=5, draft=d[np.arange(B), Lc][has_rej],
                               weights=r["weights"][np.arange(B), Lc][has_rej],
                               draft_norm=r["sigma"][np.arange(B), Lc][has_rej])
    np.testing.assert_array_equal(s["out_token"], r["out_tokens"][has_rej, L[has_rej]])
    sb = oracle.sample_residual(rows[~has_rej], L[~has_rej].astype(np.uint32), np.arange(B)[~has_rej],
                                seed=5)
    np.testing.assert_array_equal(sb["out_token"], r["out_tokens"][~has_rej, k])


def _scipy_residual_draw(l, T, d, w, sig, u):
    """The final draw of P:132 from library routines: o = scipy softmax(l / T), q = sum_n w_n d_n /
    sigma_n, r = max(0, o - q), y = the smallest v with cumsum(r)[v] > u * sum(r) (reading #10)."""
    import scipy.special
    o = scipy.special.softmax(l / T)
    q = (w[:, None] * d / sig[:, None]).sum(0)
    r = np.maximum(o - q, 0.0)
    Z = r.sum()
    return int(np.searchsorted(np.cumsum(r), u * Z, side="right")), Z


def test_sample_residual_caller_stats_branch_at_T07():
    # the caller-supplied row statistics branch (M = max l, S = sum exp((l - M) / T)) at T != 1:
    # the draw must be the one from scipy's softmax at the same T (a misplaced / T, a wrong sign or
    # a dropped normaliser moves the draw or Z)
    import scipy.special
    rng = np.random.default_rng(31)
    B, N, V, T = 64, 3, 40, 0.7
    l = rng.normal(size=(B, V)) * 2.5
    d = rng.dirichlet(np.ones(V) * 0.7, size=(B, N))
    sig = d.sum(-1)
    w = rng.dirichlet(np.ones(N), size=B)
    M = l.max(-1)
    S = np.exp(scipy.special.logsumexp(l / T, axis=-1) - M / T)
    nid = rng.integers(0, 9, size=B).astype(np.uint32)
    rid = np.arange(100, 100 + B)
    r = oracle.sample_residual(l, nid, rid, temperature=T, seed=9, step=2, row_max=M, row_sumexp=S, draft=d,
                               weights=w, draft_norm=sig)
    r0 = oracle.sample_residual(l, nid, rid, temperature=T, seed=9, step=2, draft=d, weights=w, draft_norm=sig)
    for b in range(B):
        u = oracle.uniform(9, int(rid[b]), int(nid[b]), 2, oracle.TAG_SAMPLE)
        y, Z = _scipy_residual_draw(l[b], T, d[b], w[b], sig[b], u)
        if r["tie_margin"][b] >= 1e-9:
            assert r["out_token"][b] == y, b
        assert abs(r["Z"][b] - Z) <= 1e-12 * max(1.0, Z)
    np.testing.assert_array_equal(r["out_token"], r0["out_token"])  # both branches agree
    # bonus (no drafter rows) through the caller-stats branch: a draw from softmax(l / T)
    rb = oracle.sample_residual(l, nid, rid, temperature=T, seed=9, step=2, row_max=M, row_sumexp=S)
    for b in range(B):
        u = oracle.uniform(9, int(rid[b]), int(nid[b]), 2, oracle.TAG_SAMPLE)
        o = scipy.special.softmax(l[b] / T)
        assert rb["out_token"][b] == int(np.searchsorted(np.cumsum(o), u, side="right"))


def test_sample_residual_degenerate_falls_back_to_target():
    # q == o exactly (a two-point target, a drafter row carrying the same two masses): the
    # residual has no mass, the draw falls back to o (reading #11) and is flagged
    B, V = 32, 16
    l = np.full((B, V), -np.inf)
    l[:, 3] = 0.0
    l[:, 11] = 0.0  # o = (1/2 at 3, 1/2 at 11)
    d = np.zeros((B, 1, V))
    d[:, 0, 3] = d[:, 0, 11] = 0.5
    r = oracle.sample_residual(l, np.zeros(B, np.uint32), np.arange(B), seed=4, draft=d,
                               weights=np.ones((B, 1)), draft_norm=np.ones((B, 1)))
    assert (r["status"] & oracle.INFO_DEGENERATE).all()
    for b in range(B):
        u = oracle.uniform(4, b, 0, 0, oracle.TAG_SAMPLE)
        assert r["out_token"][b] == (3 if u < 0.5 else 11)


# --------------------------------------------------------------------------- tree
def test_chain_tree_equals_linear():
    # a chain tree is the linear path, bit for bit under the same Philox stream
    rng = np.random.default_rng(13)
    B, k, N, V = 30, 4, 2, 50
    t = rng.normal(size=(B, k + 1, V)) * 3
    d = rng.dirichlet(np.ones(V) * 0.3, size=(B, k, N))
    X = np.zeros((B, k, N), np.int32)
    for b in range(B):
        for i in range(k):
            for n in range(N):
                X[b, i, n] = rng.choice(V, p=d[b, i, n])
    r = oracle.verify_batch(t, d, X, np.arange(B), seed=21)
    nn = k + 1
    parent = np.tile(np.arange(-1, k, dtype=np.int32), (B, 1))
    tok = np.zeros((B, nn), np.int32)
    tok[:, 1:] = r["fused_tokens"]
    irow = np.tile(np.array(list(range(k)) + [-1], np.int32), (B, 1))
    rt = oracle.verify_tree(parent, tok, irow, t, d, X, np.arange(B), seed=21)
    np.testing.assert_array_equal(rt["accept_len"], r["accept_len"])
    np.testing.assert_array_equal(rt["out_tokens"], r["out_tokens"])


def test_tree_enumeration_exact_and_realised():
    V, n = 3, 30000
    fan = (2, 1)
    target = _models(700, V, 3)
    drafters = [_models(800 + j, V, 3) for j in range(2)]
    law = ec.tree_law(target, drafters, fan, ec.W_CONF)
    assert sum(law.values()) == 1
    assert ec.max_tvd_to_target(law, target, V, len(fan) + 1) == 0  # reading #13 is exact
    # realisations: children drawn without replacement from the fused q (test-side)
    rng = np.random.default_rng(14)
    nn, I, N = 5, 3, 2
    parent = np.tile(np.array([-1, 0, 0, 1, 2], np.int32), (n, 1))
    irow = np.tile(np.array([0, 1, 2, -1, -1], np.int32), (n, 1))
    tok = np.zeros((n, nn), np.int32)
    t = np.zeros((n, nn, V))
    d = np.zeros((n, I, N, V))
    Xn = np.zeros((n, I, N), np.int32)

    def node(b, j, prefix, row, m):
        t[b, j] = np.log(np.array([float(x) for x in target(prefix)]))
        qs = [np.array([float(x) for x in dm(prefix)]) for dm in drafters]
        for q_i in range(N):
            d[b, row, q_i] = qs[q_i]
            Xn[b, row, q_i] = rng.choice(V, p=qs[q_i])
        c = np.array([qs[q_i][Xn[b, row, q_i]] for q_i in range(N)])
        w = c / c.sum()
        qm = w @ np.stack(qs)
        return list(rng.choice(V, size=m, replace=False, p=qm)) if m else []

    for b in range(n):
        kids = node(b, 0, (), 0, 2)
        tok[b, 1], tok[b, 2] = kids
        g1 = node(b, 1, (kids[0],), 1, 1)
        g2 = node(b, 2, (kids[1],), 2, 1)
        tok[b, 3], tok[b, 4] = g1[0], g2[0]
        t[b, 3] = np.log(np.array([float(x) for x in target((kids[0], g1[0]))]))
        t[b, 4] = np.log(np.array([float(x) for x in target((kids[1], g2[0]))]))
    rt = oracle.verify_tree(parent, tok, irow, t, d, Xn, np.arange(n), seed=99)
    assert (rt["status"] == 0).all()
    counts = {}
    for b in range(n):
        seq = tuple(int(x) for x in rt["out_tokens"][b, : rt["accept_len"][b] + 1])
        counts[seq] = counts.get(seq, 0) + 1
    assert _chi2_law(counts, law, n) > 1e-4


# ---------------- drafter-side Fuse of one iteration (NEXT-2) ----------------
def test_fuse_step_pins_against_library_routines():
    # X_n = numpy argmax (lowest index), c_n = scipy softmax at X_n, n* = first max
    import scipy.special
    rng = np.random.default_rng(3)
    B, N, V = 7, 4, 301
    l = rng.normal(size=(B, N, V)) * 3.0
    l[2, 1, 17] = l[2, 1].max() + 1.0   # a clear winner token
    l[3, 2] = l[3, 0]                   # identical drafters -> tie -> lowest n
    r = oracle.fuse_step(l, temperature=0.8)
    X = l.argmax(-1)
    p = scipy.special.softmax(l / 0.8, axis=-1)
    c = np.take_along_axis(p, X[..., None], -1)[..., 0]
    np.testing.assert_array_equal(r["own_tokens"], X)
    np.testing.assert_allclose(r["conf"], c, rtol=1e-12)
    np.testing.assert_array_equal(r["winner"], c.argmax(-1))
    np.testing.assert_array_equal(r["fused_token"], X[np.arange(B), c.argmax(-1)])
    assert (r["status"] == 0).all()
    # the closed form c = 1 / sum exp((l - max) / T)
    S = np.exp((l - l.max(-1, keepdims=True)) / 0.8).sum(-1)
    np.testing.assert_allclose(r["conf"], 1.0 / S, rtol=1e-12)


def test_fuse_step_ties_and_errors():
    l = np.zeros((3, 3, 5))
    l[0, :, 2] = 1.0                     # every drafter picks token 2 with the same confidence
    l[1, 1, 4] = 5.0                     # drafter 1 is the most confident
    l[2, 2, 0] = np.nan                  # a non-finite logit in the last drafter
    r = oracle.fuse_step(l, temperature=1.0)
    assert r["winner"][0] == 0 and r["fused_token"][0] == 2 and r["conf_gap"][0] == 0.0
    assert r["winner"][1] == 1 and r["fused_token"][1] == 4
    assert r["status"][2] == 3 and r["fused_token"][2] == -1
    # ties in a row: the lowest index is the drafter's token
    l2 = np.zeros((1, 1, 6))
    l2[0, 0, [1, 4]] = 2.0
    assert oracle.fuse_step(l2)["own_tokens"][0, 0] == 1


# ---------------- routing feedback (NEXT-3): Eqs. 1-2 ----------------
def _one_hot_emb(V, H):
    E = np.zeros((V, H))
    for v in range(V):
        E[v, v % H] = 1.0
    return E


def test_route_update_spec_examples():
    # S:273-275 (Eq. 2 evaluated by hand): c = d = 0.5 -> 0.5; K=1, c = d = 0.9 -> 0.81 / 0.82;
    # K=2 terms (0.9, 0.9) and (0.5, 0.5) -> (0.9878... + 0.5) / 2.  d is set through cosines of
    # crafted embeddings (cos = 0.9 / 0.5 between tokens 1 and 2 / 3) so that Eq. 1 feeds Eq. 2.
    H = 2
    E = np.array([[1.0, 0.0], [1.0, 0.0], [0.9, np.sqrt(1 - 0.81)], [0.5, np.sqrt(0.75)]])
    M = np.zeros((1, 1))
    r = oracle.route_update([[[2]]], [[[0.9]]], [[1]], [1], E, M)
    assert abs(r["M"][0, 0] - 0.81 / 0.82) < 1e-12 and abs(r["M"][0, 0] - 0.9878048780487805) < 1e-12
    r = oracle.route_update([[[2, 3]]], [[[0.9, 0.5]]], [[1, 1]], [2], E, M)
    assert abs(r["M"][0, 0] - 0.7439024390243902) < 1e-12
    r = oracle.route_update([[[3]]], [[[0.5]]], [[1]], [1], E, M)
    assert abs(r["M"][0, 0] - 0.5) < 1e-12


def test_route_update_eq1_cases_and_decay():
    V, H, K = 8, 8, 4
    E = _one_hot_emb(V, H)
    X = np.array([[[1, 2, 3, 4], [5, 6, 7, 0]]], np.int32)
    acc = np.array([[1, 2, 3, 4]], np.int32)
    c = np.full((1, 2, K), 0.7)
    M = np.array([[0.9, 0.9]])
    # self-similarity: the draft is the accepted prefix -> d = 1; orthogonal -> 0
    r = oracle.route_update(X, c, acc, [4], E, M)
    np.testing.assert_allclose(r["d"][0, 0], 1.0)
    np.testing.assert_allclose(r["d"][0, 1], 0.0)
    # accept_len = 0: all d = 0
    r0 = oracle.route_update(X, c, acc, [0], E, M)
    assert (r0["d"] == 0).all()
    # d beyond L is 0 (Eq. 1 "otherwise")
    r2 = oracle.route_update(X, c, acc, [2], E, M)
    np.testing.assert_allclose(r2["d"][0, 0], [1, 1, 0, 0])
    # non-participating decay: 0.5 + 0.9 (0.9 - 0.5) = 0.86
    r3 = oracle.route_update(X, c, acc, [4], E, M, participating=[[1, 0]], decay=0.9)
    assert abs(r3["M"][0, 1] - 0.86) < 1e-12
    # scores stay in (0, 1) and are monotone in c
    lo = oracle.route_update(X, np.full((1, 2, K), 0.3), acc, [3], E, M)["M"]
    hi = oracle.route_update(X, np.full((1, 2, K), 0.8), acc, [3], E, M)["M"]
    assert ((lo > 0) & (lo < 1) & (hi >= lo)).all()
    # a token outside [0, V): status 2, M unchanged
    bad = oracle.route_update(np.array([[[1, 2, 3, 99], [5, 6, 7, 0]]], np.int32), c, acc, [4], E, M)
    assert bad["status"][0] == 2 and (bad["M"] == M).all()


# ---------------- TreeSelection (NEXT-4) ----------------
def test_tree_select_spec_examples():
    # one branch, budget >= K -> a single chain; two branches diverging at step 1 ->
    # branching factor 2 under the root; budget = 1 -> the single most confident first token
    r = oracle.tree_select([[[5, 6, 7]]], [[[0.9, 0.8, 0.7]]], budget=5)
    assert r["n_nodes"][0] == 4 and list(r["parent"][0, :4]) == [-1, 0, 1, 2] and list(r["token"][0, 1:4]) == [5, 6, 7]
    r = oracle.tree_select([[[5, 6], [9, 6]]], [[[0.6, 0.9], [0.8, 0.9]]], budget=4)
    assert list(r["parent"][0, :5]) == [-1, 0, 0, 1, 2] and list(r["token"][0, 1:3]) == [9, 5]  # siblings by score
    r = oracle.tree_select([[[5, 6], [9, 6]]], [[[0.6, 0.9], [0.8, 0.9]]], budget=1)
    assert r["n_nodes"][0] == 2 and r["token"][0, 1] == 9


def _closed_best(par, sc, budget):
    # brute force: the largest total score of a prefix-closed set of `budget` non-root nodes
    import itertools
    n = len(par)
    best = -1.0
    for sub in itertools.combinations(range(1, n), min(budget, n - 1)):
        s = set(sub) | {0}
        if all(par[c] in s for c in sub):
            best = max(best, sum(sc[c] for c in sub))
    return best


def test_tree_select_is_the_best_prefix_closed_set():
    rng = np.random.default_rng(8)
    for trial in range(40):
        S, K = 3, 3
        X = rng.integers(0, 3, size=(1, S, K)).astype(np.int32)
        C = rng.uniform(0.05, 1.0, size=(1, S, K))
        full = oracle.tree_select(X, C, budget=S * K)
        n = int(full["n_nodes"][0])
        par, sc = full["parent"][0, :n], full["score"][0, :n]
        assert all(par[j] < j for j in range(1, n))                  # BFS numbering, parent first
        assert all(sc[j] <= sc[par[j]] + 1e-15 for j in range(1, n))  # scores fall along paths
        for budget in (1, 2, 4):
            r = oracle.tree_select(X, C, budget=budget)
            m = int(r["n_nodes"][0])
            assert m - 1 == min(budget, n - 1)
            assert all(r["parent"][0, j] < j for j in range(1, m))
            assert abs(r["score"][0, 1:m].sum() - _closed_best(par, sc, budget)) < 1e-12
