"""Exact rational enumeration of the verification step's output law (TEST INFRASTRUCTURE ONLY).

This is the method written as probability calculus with ``fractions.Fraction`` —
no random numbers, no floating point — so that it can pin two things:

1. what the paper fixes: speculative verification emits, at every
   reached position, a token distributed exactly as the target conditional
   o(. | prefix) ("preserving generation quality");
2. the C oracle's realisation of the same algorithm: the oracle's empirical
   output frequencies over many Philox request ids must match the exact law
   computed here (chi-square), which a dropped term, a swapped operand or a
   wrong index in either would break.

Linear drafts follow DESIGN.md §3 readings #2-#5, #10-#11; tree drafts follow
reading #13 (children drawn without replacement from the fused q, visited in
draw order, q <- q \\ {x} renormalised after each rejection).
"""
from __future__ import annotations

from fractions import Fraction
from itertools import product
from typing import Callable, Dict, List, Sequence, Tuple

Dist = List[Fraction]
W_CONF, W_WINNER, W_UNIFORM, W_POINT = 0, 1, 2, 3
SEL_ARGMAX, SEL_SAMPLE = 0, 1


def F(x) -> Fraction:
    return x if isinstance(x, Fraction) else Fraction(x)


def normalise(w: Sequence[Fraction]) -> Dist:
    z = sum(w)
    return [x / z for x in w]


def residual(p: Dist, q: Dist) -> Dist:
    """norm(max{0, p - q}); falls back to p when all mass cancels (reading #11)."""
    r = [max(Fraction(0), a - b) for a, b in zip(p, q)]
    z = sum(r)
    return p if z == 0 else [x / z for x in r]


def fusion(qs: Sequence[Dist], X: Sequence[int], weight_mode: int) -> Tuple[int, List[Fraction]]:
    """Eq. 4: n* = argmax_n q_n(X_n), ties -> lowest n; weights per reading #2."""
    c = [q[x] for q, x in zip(qs, X)]
    nstar = 0
    for n in range(1, len(c)):
        if c[n] > c[nstar]:
            nstar = n
    N = len(c)
    if weight_mode == W_CONF:
        s = sum(c)
        w = [x / s for x in c]
    elif weight_mode == W_UNIFORM:
        w = [Fraction(1, N)] * N
    else:
        w = [Fraction(int(n == nstar)) for n in range(N)]
    return nstar, w


def mix(qs: Sequence[Dist], w: Sequence[Fraction]) -> Dist:
    V = len(qs[0])
    return [sum(w[n] * qs[n][v] for n in range(len(qs))) for v in range(V)]


Model = Callable[[Tuple[int, ...]], Dist]


def linear_law(target: Model, drafters: Sequence[Model], gamma: int, weight_mode: int = W_CONF,
               select_mode: int = SEL_ARGMAX) -> Dict[Tuple[int, ...], Fraction]:
    """Exact law of the emitted token tuple of one verification round.

    Drafter n proposes X_n ~ q_n(. | fused prefix) independently (Eq. 4 conditions the
    drafters on the fused tokens x*), the fused token is Eq. 4's argmax (or a draw from the
    fused q), and the acceptance / residual / bonus rules are P:130-133.
    """
    law: Dict[Tuple[int, ...], Fraction] = {}

    def rec(prefix: Tuple[int, ...], i: int, prob: Fraction):
        p = target(prefix)
        V = len(p)
        if i == gamma:  # all accepted: bonus x_{gamma+1} ~ o
            for y in range(V):
                if p[y]:
                    law[prefix + (y,)] = law.get(prefix + (y,), 0) + prob * p[y]
            return
        qs = [d(prefix) for d in drafters]
        for X in product(range(V), repeat=len(qs)):
            px = prob
            for n, x in enumerate(X):
                px *= qs[n][x]
            if px == 0:
                continue
            nstar, w = fusion(qs, X, weight_mode)
            qmix = mix(qs, w)
            cands = [(X[nstar], Fraction(1))] if select_mode == SEL_ARGMAX else \
                [(x, qmix[x]) for x in range(V) if qmix[x]]
            for xs, pxs in cands:
                q = qmix if weight_mode != W_POINT else [Fraction(int(v == xs)) for v in range(V)]
                a = min(Fraction(1), p[xs] / q[xs])  # accept with min(1, o/q)
                base = px * pxs
                if a:
                    rec(prefix + (xs,), i + 1, base * a)
                if a != 1:  # reject -> resample from norm(max(0, o - q)) and stop
                    r = residual(p, q)
                    for y in range(V):
                        if r[y]:
                            key = prefix + (y,)
                            law[key] = law.get(key, 0) + base * (1 - a) * r[y]

    rec((), 0, Fraction(1))
    return law


def tree_law(target: Model, drafters: Sequence[Model], fanout: Sequence[int],
             weight_mode: int = W_CONF) -> Dict[Tuple[int, ...], Fraction]:
    """Exact law of the emitted tokens for a tree whose depth-d nodes have fanout[d] children,
    drawn without replacement from the fused q at the parent and visited in draw order
    (reading #13).  Leaves are at depth len(fanout)."""
    law: Dict[Tuple[int, ...], Fraction] = {}

    def sample_children(q: Dist, m: int):
        """Ordered draws without replacement: yields (tuple, probability)."""
        V = len(q)

        def r(chosen, mass_left, prob):
            if len(chosen) == m:
                yield tuple(chosen), prob
                return
            for x in range(V):
                if x in chosen or q[x] == 0:
                    continue
                yield from r(chosen + [x], mass_left - q[x], prob * q[x] / mass_left)

        yield from r([], Fraction(1), Fraction(1))

    def emit(key, pr):
        law[key] = law.get(key, 0) + pr

    def rec(prefix: Tuple[int, ...], depth: int, prob: Fraction):
        p = target(prefix)
        V = len(p)
        if depth == len(fanout):
            for y in range(V):
                if p[y]:
                    emit(prefix + (y,), prob * p[y])
            return
        qs = [d(prefix) for d in drafters]
        for X in product(range(V), repeat=len(qs)):
            px = prob
            for n, x in enumerate(X):
                px *= qs[n][x]
            if px == 0:
                continue
            _, w = fusion(qs, X, weight_mode)
            q0 = mix(qs, w)
            m = min(fanout[depth], sum(1 for v in q0 if v))
            for kids, pk in sample_children(q0, m):
                walk(prefix, depth, p, q0, kids, px * pk)

    def walk(prefix, depth, p, q, kids, prob):
        V = len(p)
        if not kids:  # children exhausted: y ~ current p
            for y in range(V):
                if p[y]:
                    emit(prefix + (y,), prob * p[y])
            return
        x = kids[0]
        a = min(Fraction(1), p[x] / q[x])
        if a:
            rec(prefix + (x,), depth + 1, prob * a)
        if a != 1:
            p2 = residual(p, q)
            q2 = [Fraction(0) if v == x else q[v] / (1 - q[x]) for v in range(V)] if q[x] != 1 else q
            walk(prefix, depth, p2, q2, kids[1:], prob * (1 - a))

    rec((), 0, Fraction(1))
    return law


def position_conditionals(law: Dict[Tuple[int, ...], Fraction], j: int, V: int):
    """For every prefix a_<j reached with positive probability, the law of the token emitted at
    position j given the prefix and that position j is emitted."""
    acc: Dict[Tuple[int, ...], List[Fraction]] = {}
    for seq, pr in law.items():
        if len(seq) > j:
            acc.setdefault(seq[:j], [Fraction(0)] * V)[seq[j]] += pr
    return {pre: normalise(v) for pre, v in acc.items()}


def max_tvd_to_target(law, target: Model, V: int, depth: int) -> Fraction:
    """max over positions j < depth and reached prefixes of TV(emitted_j | prefix, o(.|prefix))."""
    worst = Fraction(0)
    for j in range(depth):
        for pre, dist in position_conditionals(law, j, V).items():
            o = target(pre)
            tv = sum(abs(a - b) for a, b in zip(dist, o)) / 2
            worst = max(worst, tv)
    return worst


def expected_first_acceptance(p: Dist, q: Dist) -> Fraction:
    """Closed form P(accept x ~ q) = sum_v min(p(v), q(v)) (follows from P:130-131)."""
    return sum(min(a, b) for a, b in zip(p, q))


def random_dist(rng, V: int, zeros: bool = False) -> Dist:
    w = [Fraction(int(rng.integers(0 if zeros else 1, 7))) for _ in range(V)]
    if sum(w) == 0:
        w[int(rng.integers(0, V))] = Fraction(1)
    return normalise(w)


def random_tabular_model(rng, V: int, depth: int, zeros: bool = False) -> Model:
    """A context-dependent toy model over prefixes of length <= depth (S:107-117 style)."""
    table: Dict[Tuple[int, ...], Dist] = {}

    def m(prefix: Tuple[int, ...]) -> Dist:
        if prefix not in table:
            table[prefix] = random_dist(rng, V, zeros)
        return table[prefix]

    return m
