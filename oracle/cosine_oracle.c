/*
 * cosine_oracle.c — TEST INFRASTRUCTURE ONLY (see cosine_oracle.h).
 *
 * A plain, slow, obviously correct fp64 implementation of the verification
 * step of CoSine (arXiv 2503.10325), written from the paper:
 *   - acceptance test, first rejection, residual resample, bonus token:
 *     §2.1, PAPER.md P:130-133;
 *   - confidence-based token fusion: Eq. 4; confidence c = P(x): P:311-314;
 *   - batched "foreach draft in parallel: Verify": Alg. 2, P:463-464;
 *   - tree-shaped drafts: P:134, P:414-415 (algorithm = DESIGN.md reading #13).
 * Where the paper is silent the DESIGN.md readings (#1-#18) are cited.
 *
 * Every loop runs in ascending index order, every sum is a sequential fp64
 * sum, nothing is blocked or fused.  Compiled with -O2 -ffp-contract=off.
 */
#include "cosine_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), reading #8.      */
/* ------------------------------------------------------------------ */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
    uint64_t prod0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
    uint64_t prod1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
    uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* U(rid, node, tag) = (x0 >> 8) * 2^-24, ctr = {rid_lo, rid_hi, node, (step<<4)|tag},
 * key = {seed_lo, seed_hi}  (readings #8, #9). */
double orc_uniform(uint64_t seed, uint64_t request_id, uint32_t node, uint32_t step, uint32_t tag) {
  uint32_t ctr[4] = {(uint32_t)request_id, (uint32_t)(request_id >> 32), node, (step << 4) | tag};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  orc_philox4x32_10(ctr, key, out);
  return (double)(out[0] >> 8) * (1.0 / 16777216.0);
}

/* ------------------------------------------------------------------ */
/* Distributions                                                       */
/* ------------------------------------------------------------------ */

/* Inverse CDF, reading #10: smallest v (ascending index) with C(v) = sum_{w<=v} w(w) > t,
 * t = u * Z; if none (rounding), the last v with w(v) > 0. */
int64_t orc_invcdf(const double* w, int64_t V, double u, double* margin) {
  double Z = 0.0;
  for (int64_t v = 0; v < V; ++v) Z += w[v];
  double t = u * Z;
  double C = 0.0;
  for (int64_t v = 0; v < V; ++v) {
    double Cprev = C;
    C += w[v];
    if (C > t) {
      if (margin) {
        double a = t - Cprev, b = C - t;
        *margin = (a < b ? a : b) / Z;
      }
      return v;
    }
  }
  for (int64_t v = V - 1; v >= 0; --v)
    if (w[v] > 0.0) {
      if (margin) *margin = 0.0;
      return v;
    }
  if (margin) *margin = 0.0;
  return -1;
}

/* o_i(x) as a probability vector (reading #1): p = softmax(l / T), T > 0.
 * +inf / NaN logits are non-finite input; all -inf is an empty row. */
int orc_softmax(const double* l, int64_t V, double T, double* p, double* M, double* S) {
  for (int64_t v = 0; v < V; ++v)
    if (isnan(l[v]) || (isinf(l[v]) && l[v] > 0)) return ORC_ST_NONFINITE_OR_NEGATIVE;
  double m = -INFINITY;
  for (int64_t v = 0; v < V; ++v) {
    double z = l[v] / T;
    if (z > m) m = z;
  }
  if (m == -INFINITY) return ORC_ST_EMPTY_ROW;
  double s = 0.0;
  for (int64_t v = 0; v < V; ++v) s += exp(l[v] / T - m);
  for (int64_t v = 0; v < V; ++v) p[v] = exp(l[v] / T - m) / s;
  if (M) *M = m;
  if (S) *S = s;
  return 0;
}

/* Greedy (T = 0, reading #7): lowest-index argmax. */
static int orc_argmax(const double* l, int64_t V, int64_t* am) {
  for (int64_t v = 0; v < V; ++v)
    if (isnan(l[v]) || (isinf(l[v]) && l[v] > 0)) return ORC_ST_NONFINITE_OR_NEGATIVE;
  int64_t best = -1;
  double bv = -INFINITY;
  for (int64_t v = 0; v < V; ++v)
    if (l[v] > bv) { bv = l[v]; best = v; }
  if (best < 0) return ORC_ST_EMPTY_ROW;
  *am = best;
  return 0;
}

/* norm(max{0, o - q}).  Returns 1 when all mass cancels. */
int orc_residual(const double* o, const double* q, int64_t V, double* r) {
  double Z = 0.0;
  for (int64_t v = 0; v < V; ++v) {
    double d = o[v] - q[v];
    r[v] = d > 0.0 ? d : 0.0;
    Z += r[v];
  }
  if (Z == 0.0) return 1;
  for (int64_t v = 0; v < V; ++v) r[v] /= Z;
  return 0;
}

/* Drafter distribution q_n (reading #6): PROBS rows are renormalised by their sum
 * (sigma); LOGITS rows are softmax(d / T).  Returns status; sigma = sum (PROBS) or
 * sum-exp (LOGITS, max-shifted). */
static int orc_draft_dist(const double* d, int64_t V, int32_t kind, double T, double* q,
                          double* sigma) {
  if (kind == ORC_DRAFT_PROBS) {
    for (int64_t v = 0; v < V; ++v)
      if (isnan(d[v]) || isinf(d[v]) || d[v] < 0.0) return ORC_ST_NONFINITE_OR_NEGATIVE;
    double s = 0.0;
    for (int64_t v = 0; v < V; ++v) s += d[v];
    if (s == 0.0) return ORC_ST_EMPTY_ROW;
    for (int64_t v = 0; v < V; ++v) q[v] = d[v] / s;
    *sigma = s;
    return 0;
  }
  double M, S;
  int st = orc_softmax(d, V, T, q, &M, &S);
  *sigma = S;
  return st;
}

/* Eq. 4 with ties -> lowest drafter index (reading #5),
 * then the weights of the fused distribution (reading #2). */
static int orc_fusion_weights(int32_t N, const double* c, int32_t weight_mode, double* w,
                              double* gap) {
  int nstar = 0;
  for (int n = 1; n < N; ++n)
    if (c[n] > c[nstar]) nstar = n;
  /* relative gap between the best and second best confidence (reading #18) */
  double second = -1.0;
  for (int n = 0; n < N; ++n)
    if (n != nstar && c[n] > second) second = c[n];
  *gap = (N > 1) ? (c[nstar] - second) / c[nstar] : 1.0;
  if (weight_mode == ORC_W_CONF) {
    double sc = 0.0;
    for (int n = 0; n < N; ++n) sc += c[n];
    for (int n = 0; n < N; ++n) w[n] = c[n] / sc;
  } else if (weight_mode == ORC_W_UNIFORM) {
    for (int n = 0; n < N; ++n) w[n] = 1.0 / (double)N;
  } else { /* WINNER, POINT: one-hot on n* */
    for (int n = 0; n < N; ++n) w[n] = (n == nstar) ? 1.0 : 0.0;
  }
  return nstar;
}

static double dmin(double a, double b) { return a < b ? a : b; }

/* ------------------------------------------------------------------ */
/* Linear verification (§8(c) steps 1-7)                               */
/* ------------------------------------------------------------------ */
int orc_verify_batch(int32_t B, int32_t k, int32_t N, int64_t V,
                     const double* target, double T,
                     const double* draft, int32_t draft_kind,
                     const int32_t* draft_tokens, const int32_t* draft_len,
                     const uint64_t* request_ids, uint64_t seed, uint32_t step,
                     int32_t weight_mode, int32_t select_mode,
                     int32_t* accept_len, int32_t* out_tokens, int32_t* status,
                     double* dbg_p_x, double* dbg_q_x, double* dbg_M, double* dbg_S,
                     double* dbg_sigma, double* dbg_conf, double* dbg_w, int32_t* dbg_fused,
                     double* dbg_u, double* dbg_Z, double* tie_margin) {
  if (B < 0 || k < 1 || N < 1 || N > 8 || V < 1 || T < 0.0) return 1;
  if (weight_mode < 0 || weight_mode > 3 || select_mode < 0 || select_mode > 1) return 1;
  if (weight_mode == ORC_W_POINT && select_mode == ORC_SEL_SAMPLE) return 1;
  if (T == 0.0 && (draft_kind == ORC_DRAFT_LOGITS || select_mode == ORC_SEL_SAMPLE)) return 1;
  const int greedy = (T == 0.0);

  double* p = (double*)malloc(sizeof(double) * (size_t)(k + 1) * (size_t)V);   /* p_i rows */
  double* qn = (double*)malloc(sizeof(double) * (size_t)N * (size_t)V);        /* q_{n,i} */
  double* qf = (double*)malloc(sizeof(double) * (size_t)k * (size_t)V);        /* fused q_i */
  double* r = (double*)malloc(sizeof(double) * (size_t)V);
  int64_t* amax = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k + 1));
  int32_t* xstar = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  double* pxs = (double*)malloc(sizeof(double) * (size_t)k);
  double* qxs = (double*)malloc(sizeof(double) * (size_t)k);
  double* margin_acc = (double*)malloc(sizeof(double) * (size_t)k);
  double* margin_fuse = (double*)malloc(sizeof(double) * (size_t)k);
  int* acc = (int*)malloc(sizeof(int) * (size_t)k);
  if (!p || !qn || !qf || !r || !amax || !xstar || !pxs || !qxs || !margin_acc || !margin_fuse || !acc) {
    free(p); free(qn); free(qf); free(r); free(amax); free(xstar); free(pxs); free(qxs);
    free(margin_acc); free(margin_fuse); free(acc);
    return 1;
  }

  for (int32_t b = 0; b < B; ++b) {
    const uint64_t rid = request_ids[b];
    int32_t* out = out_tokens + (size_t)b * (size_t)(k + 1);
    for (int j = 0; j <= k; ++j) out[j] = -1;
    accept_len[b] = -1;
    status[b] = ORC_ST_OK;
    if (tie_margin) tie_margin[b] = INFINITY;
    if (dbg_Z) dbg_Z[b] = NAN;
    const int32_t g = draft_len ? draft_len[b] : k; /* gamma_b, reading #15 */
    if (g < 1 || g > k) { status[b] = ORC_ST_BAD_DRAFT_LEN; continue; }

    int err = 0;
    double tm = INFINITY;
    /* Steps 1-4 for every position i in [0, g]; the first unit (position) with an error
     * decides the request's status (reading #12, precedence 2 > 3 > 4 > 1 within a unit). */
    for (int32_t i = 0; i <= g && !err; ++i) {
      const double* l = target + ((size_t)b * (size_t)(k + 1) + (size_t)i) * (size_t)V;
      double* pi = p + (size_t)i * (size_t)V;
      int e_tok = 0, e_nf = 0, e_empty = 0, e_zero = 0;
      /* step 1: target distribution */
      double M = NAN, S = NAN;
      int st;
      if (greedy) {
        st = orc_argmax(l, V, &amax[i]);
        if (!st) {
          for (int64_t v = 0; v < V; ++v) pi[v] = 0.0;
          pi[amax[i]] = 1.0;
          M = l[amax[i]];
        }
      } else {
        st = orc_softmax(l, V, T, pi, &M, &S);
      }
      if (st == ORC_ST_NONFINITE_OR_NEGATIVE) e_nf = 1;
      if (st == ORC_ST_EMPTY_ROW) e_empty = 1;
      if (dbg_M) dbg_M[(size_t)b * (size_t)(k + 1) + (size_t)i] = M;
      if (dbg_S) dbg_S[(size_t)b * (size_t)(k + 1) + (size_t)i] = S;
      if (i < g) {
        const int32_t* X = draft_tokens + ((size_t)b * (size_t)k + (size_t)i) * (size_t)N;
        for (int n = 0; n < N; ++n)
          if (X[n] < 0 || (int64_t)X[n] >= V) e_tok = 1;
        double sigma[8], c[8], w[8];
        for (int n = 0; n < N; ++n) {
          const double* d = draft + (((size_t)b * (size_t)k + (size_t)i) * (size_t)N + (size_t)n) * (size_t)V;
          int sd = orc_draft_dist(d, V, draft_kind, T, qn + (size_t)n * (size_t)V, &sigma[n]);
          if (sd == ORC_ST_NONFINITE_OR_NEGATIVE) e_nf = 1;
          if (sd == ORC_ST_EMPTY_ROW) e_empty = 1;
        }
        if (!e_tok && !e_nf && !e_empty) {
          /* step 3: confidences c_{n,i} = q_{n,i}(X_{n,i})  (reading #4) */
          for (int n = 0; n < N; ++n) {
            c[n] = qn[(size_t)n * (size_t)V + (size_t)X[n]];
            if (c[n] == 0.0) e_zero = 1;
          }
        }
        if (!e_tok && !e_nf && !e_empty && !e_zero) {
          /* step 4: fusion (Eq. 4) and the fused distribution q_i (reading #2) */
          double gap;
          int nstar = orc_fusion_weights(N, c, weight_mode, w, &gap);
          double* qi = qf + (size_t)i * (size_t)V;
          for (int64_t v = 0; v < V; ++v) {
            double s = 0.0;
            for (int n = 0; n < N; ++n) s += w[n] * qn[(size_t)n * (size_t)V + (size_t)v];
            qi[v] = s;
          }
          double mf = (select_mode == ORC_SEL_ARGMAX) ? gap : INFINITY;
          if (select_mode == ORC_SEL_ARGMAX) {
            xstar[i] = X[nstar];
          } else {
            double m2;
            double uf = orc_uniform(seed, rid, (uint32_t)(i + 1), step, ORC_TAG_FUSE);
            xstar[i] = (int32_t)orc_invcdf(qi, V, uf, &m2);
            mf = dmin(mf, m2);
          }
          if (weight_mode == ORC_W_POINT) {
            for (int64_t v = 0; v < V; ++v) qi[v] = 0.0;
            qi[xstar[i]] = 1.0;
          }
          margin_fuse[i] = mf;
          pxs[i] = pi[xstar[i]];
          qxs[i] = qi[xstar[i]];
          if (dbg_fused) dbg_fused[(size_t)b * (size_t)k + (size_t)i] = xstar[i];
          for (int n = 0; n < N; ++n) {
            size_t o = ((size_t)b * (size_t)k + (size_t)i) * (size_t)N + (size_t)n;
            if (dbg_sigma) dbg_sigma[o] = sigma[n];
            if (dbg_conf) dbg_conf[o] = c[n];
            if (dbg_w) dbg_w[o] = w[n];
          }
        }
      }
      if (e_tok) err = ORC_ST_TOKEN_OUT_OF_RANGE;
      else if (e_nf) err = ORC_ST_NONFINITE_OR_NEGATIVE;
      else if (e_empty) err = ORC_ST_EMPTY_ROW;
      else if (e_zero) err = ORC_ST_ZERO_PROB_DRAFT;
    }
    if (err) { status[b] = err; continue; }

    /* step 5: acceptance u * q(x*) < p(x*), i.e. u < min(1, p/q) (reading #9);
     * first rejection. */
    int32_t L = g;
    for (int32_t i = 0; i < g; ++i) {
      double u = orc_uniform(seed, rid, (uint32_t)(i + 1), step, ORC_TAG_ACCEPT);
      if (dbg_u) dbg_u[(size_t)b * (size_t)k + (size_t)i] = u;
      if (greedy) {
        acc[i] = ((int64_t)xstar[i] == amax[i]);
        margin_acc[i] = INFINITY;
      } else {
        acc[i] = (u * qxs[i] < pxs[i]);
        margin_acc[i] = fabs(u - pxs[i] / qxs[i]);
      }
      if (dbg_p_x) dbg_p_x[(size_t)b * (size_t)k + (size_t)i] = pxs[i];
      if (dbg_q_x) dbg_q_x[(size_t)b * (size_t)k + (size_t)i] = qxs[i];
    }
    for (int32_t i = 0; i < g; ++i)
      if (!acc[i]) { L = i; break; }
    for (int32_t i = 0; i < g && i <= L; ++i) {
      if (i < L || !acc[i]) tm = dmin(tm, margin_acc[i]);
      tm = dmin(tm, margin_fuse[i]);
    }

    /* step 6: the final token */
    int64_t y;
    const double* pL = p + (size_t)L * (size_t)V;
    if (greedy) {
      y = amax[L];
    } else {
      double us = orc_uniform(seed, rid, (uint32_t)L, step, ORC_TAG_SAMPLE);
      double ms;
      if (L < g) {
        const double* qL = qf + (size_t)L * (size_t)V;
        double Z = 0.0;
        for (int64_t v = 0; v < V; ++v) {
          double d = pL[v] - qL[v];
          r[v] = d > 0.0 ? d : 0.0;
          Z += r[v];
        }
        if (Z == 0.0) { /* reading #11: fall back to p */
          status[b] |= ORC_INFO_DEGENERATE_RESIDUAL;
          for (int64_t v = 0; v < V; ++v) r[v] = pL[v];
          Z = 1.0;
        }
        if (dbg_Z) dbg_Z[b] = Z;
        y = orc_invcdf(r, V, us, &ms);
      } else {
        if (dbg_Z) dbg_Z[b] = 1.0;
        y = orc_invcdf(pL, V, us, &ms);
      }
      tm = dmin(tm, ms);
    }
    /* step 7: emit x*_0 .. x*_{L-1}, y */
    for (int32_t i = 0; i < L; ++i) out[i] = xstar[i];
    out[L] = (int32_t)y;
    accept_len[b] = L;
    if (tie_margin) tie_margin[b] = tm;
  }
  free(p); free(qn); free(qf); free(r); free(amax); free(xstar); free(pxs); free(qxs);
  free(margin_acc); free(margin_fuse); free(acc);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Fusion only (Eq. 4)                                                 */
/* ------------------------------------------------------------------ */
int orc_fuse_drafts(int32_t B, int32_t k, int32_t N, int64_t V,
                    const double* draft, int32_t draft_kind, double T,
                    const int32_t* draft_tokens, const uint64_t* request_ids,
                    uint64_t seed, uint32_t step, int32_t weight_mode, int32_t select_mode,
                    int32_t* fused_tokens, double* weights, double* draft_norm,
                    double* fused_q, int32_t* status, double* tie_margin) {
  if (B < 0 || k < 1 || N < 1 || N > 8 || V < 1) return 1;
  if (weight_mode < 0 || weight_mode > 3 || select_mode < 0 || select_mode > 1) return 1;
  if (weight_mode == ORC_W_POINT && select_mode == ORC_SEL_SAMPLE) return 1;
  if (draft_kind == ORC_DRAFT_LOGITS && !(T > 0.0)) return 1;
  double* qn = (double*)malloc(sizeof(double) * (size_t)N * (size_t)V);
  double* qi = (double*)malloc(sizeof(double) * (size_t)V);
  if (!qn || !qi) { free(qn); free(qi); return 1; }
  for (int32_t b = 0; b < B; ++b) {
    status[b] = 0;
    double tm = INFINITY;
    int err = 0;
    for (int32_t i = 0; i < k; ++i) {
      fused_tokens[(size_t)b * (size_t)k + (size_t)i] = -1;
      if (err) continue;
      const int32_t* X = draft_tokens + ((size_t)b * (size_t)k + (size_t)i) * (size_t)N;
      int e_tok = 0, e_nf = 0, e_empty = 0, e_zero = 0;
      double sigma[8], c[8], w[8];
      for (int n = 0; n < N; ++n)
        if (X[n] < 0 || (int64_t)X[n] >= V) e_tok = 1;
      for (int n = 0; n < N; ++n) {
        const double* d = draft + (((size_t)b * (size_t)k + (size_t)i) * (size_t)N + (size_t)n) * (size_t)V;
        int sd = orc_draft_dist(d, V, draft_kind, T, qn + (size_t)n * (size_t)V, &sigma[n]);
        if (sd == ORC_ST_NONFINITE_OR_NEGATIVE) e_nf = 1;
        if (sd == ORC_ST_EMPTY_ROW) e_empty = 1;
      }
      if (!e_tok && !e_nf && !e_empty)
        for (int n = 0; n < N; ++n) {
          c[n] = qn[(size_t)n * (size_t)V + (size_t)X[n]];
          if (c[n] == 0.0) e_zero = 1;
        }
      if (e_tok) err = ORC_ST_TOKEN_OUT_OF_RANGE;
      else if (e_nf) err = ORC_ST_NONFINITE_OR_NEGATIVE;
      else if (e_empty) err = ORC_ST_EMPTY_ROW;
      else if (e_zero) err = ORC_ST_ZERO_PROB_DRAFT;
      if (err) continue;
      double gap;
      int nstar = orc_fusion_weights(N, c, weight_mode, w, &gap);
      for (int64_t v = 0; v < V; ++v) {
        double s = 0.0;
        for (int n = 0; n < N; ++n) s += w[n] * qn[(size_t)n * (size_t)V + (size_t)v];
        qi[v] = s;
      }
      int32_t xs;
      if (select_mode == ORC_SEL_ARGMAX) {
        xs = X[nstar];
        tm = dmin(tm, gap);
      } else {
        double m2;
        double uf = orc_uniform(seed, request_ids[b], (uint32_t)(i + 1), step, ORC_TAG_FUSE);
        xs = (int32_t)orc_invcdf(qi, V, uf, &m2);
        tm = dmin(tm, m2);
      }
      if (weight_mode == ORC_W_POINT) {
        for (int64_t v = 0; v < V; ++v) qi[v] = 0.0;
        qi[xs] = 1.0;
      }
      fused_tokens[(size_t)b * (size_t)k + (size_t)i] = xs;
      for (int n = 0; n < N; ++n) {
        size_t o = ((size_t)b * (size_t)k + (size_t)i) * (size_t)N + (size_t)n;
        if (weights) weights[o] = w[n];
        if (draft_norm) draft_norm[o] = sigma[n];
      }
      if (fused_q)
        for (int64_t v = 0; v < V; ++v)
          fused_q[((size_t)b * (size_t)k + (size_t)i) * (size_t)V + (size_t)v] = qi[v];
    }
    if (err) {
      status[b] = err;
      for (int32_t i = 0; i < k; ++i) fused_tokens[(size_t)b * (size_t)k + (size_t)i] = -1;
    }
    if (tie_margin) tie_margin[b] = tm;
  }
  free(qn); free(qi);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Residual / bonus sample of one row group                */
/* ------------------------------------------------------------------ */
int orc_sample_residual(int32_t B, int64_t V, const double* target, double T,
                        const double* row_max, const double* row_sumexp,
                        const double* draft, int32_t N, const double* weights,
                        const double* draft_norm, const uint32_t* node_ids,
                        const uint64_t* request_ids, uint64_t seed, uint32_t step,
                        int32_t* out_token, int32_t* status, double* dbg_Z, double* tie_margin) {
  if (B < 0 || V < 1 || T < 0.0) return 1;
  if (draft && (N < 1 || N > 8 || !weights || !draft_norm)) return 1;
  if ((row_max == NULL) != (row_sumexp == NULL)) return 1;
  double* p = (double*)malloc(sizeof(double) * (size_t)V);
  double* r = (double*)malloc(sizeof(double) * (size_t)V);
  if (!p || !r) { free(p); free(r); return 1; }
  for (int32_t b = 0; b < B; ++b) {
    const double* l = target + (size_t)b * (size_t)V;
    out_token[b] = -1;
    status[b] = 0;
    if (tie_margin) tie_margin[b] = INFINITY;
    if (dbg_Z) dbg_Z[b] = NAN;
    int st = 0;
    if (T == 0.0) {
      int64_t am;
      st = orc_argmax(l, V, &am);
      if (st) { status[b] = st; continue; }
      out_token[b] = (int32_t)am;
      continue;
    }
    if (row_max) {
      /* caller-provided stats: M = max_v l(v) (raw logit), S = sum exp((l - M)/T) */
      for (int64_t v = 0; v < V; ++v)
        if (isnan(l[v]) || (isinf(l[v]) && l[v] > 0)) st = ORC_ST_NONFINITE_OR_NEGATIVE;
      if (!st && !(row_sumexp[b] > 0.0)) st = ORC_ST_EMPTY_ROW;
      if (!st)
        for (int64_t v = 0; v < V; ++v) p[v] = exp((l[v] - row_max[b]) / T) / row_sumexp[b];
    } else {
      st = orc_softmax(l, V, T, p, NULL, NULL);
    }
    if (!st && draft) {
      for (int n = 0; n < N && !st; ++n) {
        const double* d = draft + ((size_t)b * (size_t)N + (size_t)n) * (size_t)V;
        for (int64_t v = 0; v < V; ++v)
          if (isnan(d[v]) || isinf(d[v]) || d[v] < 0.0) st = ORC_ST_NONFINITE_OR_NEGATIVE;
        if (!st && !(draft_norm[(size_t)b * (size_t)N + (size_t)n] > 0.0)) st = ORC_ST_EMPTY_ROW;
      }
    }
    if (st) { status[b] = st; continue; }
    double u = orc_uniform(seed, request_ids[b], node_ids[b], step, ORC_TAG_SAMPLE);
    double Z = 1.0, ms;
    if (draft) {
      Z = 0.0;
      for (int64_t v = 0; v < V; ++v) {
        double q = 0.0;
        for (int n = 0; n < N; ++n)
          q += weights[(size_t)b * (size_t)N + (size_t)n] *
               (draft[((size_t)b * (size_t)N + (size_t)n) * (size_t)V + (size_t)v] /
                draft_norm[(size_t)b * (size_t)N + (size_t)n]);
        double d = p[v] - q;
        r[v] = d > 0.0 ? d : 0.0;
        Z += r[v];
      }
      if (Z == 0.0) {
        status[b] |= ORC_INFO_DEGENERATE_RESIDUAL;
        for (int64_t v = 0; v < V; ++v) r[v] = p[v];
        Z = 1.0;
      }
      out_token[b] = (int32_t)orc_invcdf(r, V, u, &ms);
    } else {
      out_token[b] = (int32_t)orc_invcdf(p, V, u, &ms);
    }
    if (dbg_Z) dbg_Z[b] = Z;
    if (tie_margin) tie_margin[b] = ms;
  }
  free(p); free(r);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Tree verification: multi-candidate recursive rejection, children     */
/* visited in slot order, q <- q \ {x} renormalised (reading #13).     */
/* ------------------------------------------------------------------ */
int orc_verify_tree(int32_t B, int32_t J, int32_t I, int32_t N, int64_t V,
                    const int32_t* parent, const int32_t* node_token, const int32_t* internal_row,
                    const double* target, double T,
                    const double* draft, int32_t draft_kind, const int32_t* node_draft_tokens,
                    const uint64_t* request_ids, uint64_t seed, uint32_t step, int32_t weight_mode,
                    int32_t* accept_len, int32_t* accepted_nodes, int32_t* out_tokens,
                    int32_t* status, double* tie_margin) {
  if (B < 0 || J < 0 || I < 0 || N < 1 || N > 8 || V < 1 || !(T > 0.0)) return 1;
  if (weight_mode < 0 || weight_mode > 2) return 1; /* POINT undefined for multi-child nodes */
  const int32_t nn = J + 1;
  double* p = (double*)malloc(sizeof(double) * (size_t)V);
  double* q = (double*)malloc(sizeof(double) * (size_t)V);
  double* r = (double*)malloc(sizeof(double) * (size_t)V);
  double* qn = (double*)malloc(sizeof(double) * (size_t)N * (size_t)V);
  if (!p || !q || !r || !qn) { free(p); free(q); free(r); free(qn); return 1; }
  for (int32_t b = 0; b < B; ++b) {
    const int32_t* par = parent + (size_t)b * (size_t)nn;
    const int32_t* tok = node_token + (size_t)b * (size_t)nn;
    const int32_t* irow = internal_row + (size_t)b * (size_t)nn;
    const uint64_t rid = request_ids[b];
    int32_t* an = accepted_nodes + (size_t)b * (size_t)nn;
    int32_t* out = out_tokens + (size_t)b * (size_t)nn;
    for (int j = 0; j < nn; ++j) { an[j] = -1; out[j] = -1; }
    accept_len[b] = -1;
    status[b] = 0;
    if (tie_margin) tie_margin[b] = INFINITY;
    /* structure: parent[0] = -1, 0 <= parent[j] < j; tokens in range; distinct sibling
     * tokens; internal_row set exactly for nodes with children. */
    int err = 0;
    if (par[0] != -1) err = ORC_ST_BAD_TREE;
    for (int j = 1; j < nn && !err; ++j) {
      if (par[j] < 0 || par[j] >= j) err = ORC_ST_BAD_TREE;
      else if (tok[j] < 0 || (int64_t)tok[j] >= V) err = ORC_ST_TOKEN_OUT_OF_RANGE;
      for (int j2 = 1; j2 < j && !err; ++j2)
        if (par[j2] == par[j] && tok[j2] == tok[j]) err = ORC_ST_BAD_TREE;
    }
    for (int j = 0; j < nn && !err; ++j) {
      int has_child = 0;
      for (int c = j + 1; c < nn; ++c) if (par[c] == j) has_child = 1;
      if (has_child != (irow[j] >= 0) || irow[j] >= I) err = ORC_ST_BAD_TREE;
    }
    /* all-node validation in node order (every row of the request is input) */
    for (int j = 0; j < nn && !err; ++j) {
      const double* l = target + ((size_t)b * (size_t)nn + (size_t)j) * (size_t)V;
      int st = orc_softmax(l, V, T, p, NULL, NULL);
      int e_tok = 0, e_nf = (st == ORC_ST_NONFINITE_OR_NEGATIVE), e_empty = (st == ORC_ST_EMPTY_ROW), e_zero = 0;
      if (irow[j] >= 0) {
        const int32_t* X = node_draft_tokens + ((size_t)b * (size_t)I + (size_t)irow[j]) * (size_t)N;
        for (int n = 0; n < N; ++n) if (X[n] < 0 || (int64_t)X[n] >= V) e_tok = 1;
        double sigma;
        for (int n = 0; n < N; ++n) {
          const double* d = draft + (((size_t)b * (size_t)I + (size_t)irow[j]) * (size_t)N + (size_t)n) * (size_t)V;
          int sd = orc_draft_dist(d, V, draft_kind, T, qn + (size_t)n * (size_t)V, &sigma);
          if (sd == ORC_ST_NONFINITE_OR_NEGATIVE) e_nf = 1;
          if (sd == ORC_ST_EMPTY_ROW) e_empty = 1;
        }
        if (!e_tok && !e_nf && !e_empty) {
          for (int n = 0; n < N; ++n) if (qn[(size_t)n * (size_t)V + (size_t)X[n]] == 0.0) e_zero = 1;
          if (!e_zero) {
            double c[8], w[8], gap;
            for (int n = 0; n < N; ++n) c[n] = qn[(size_t)n * (size_t)V + (size_t)X[n]];
            orc_fusion_weights(N, c, weight_mode, w, &gap);
            for (int c2 = j + 1; c2 < nn; ++c2)
              if (par[c2] == j) {
                double qx = 0.0;
                for (int n = 0; n < N; ++n) qx += w[n] * qn[(size_t)n * (size_t)V + (size_t)tok[c2]];
                if (qx == 0.0) e_zero = 1;
              }
          }
        }
      }
      if (e_tok) err = ORC_ST_TOKEN_OUT_OF_RANGE;
      else if (e_nf) err = ORC_ST_NONFINITE_OR_NEGATIVE;
      else if (e_empty) err = ORC_ST_EMPTY_ROW;
      else if (e_zero) err = ORC_ST_ZERO_PROB_DRAFT;
    }
    if (err) { status[b] = err; continue; }

    /* the walk; the current target distribution is p = pw / pz so that a chain tree
     * performs exactly the arithmetic of the linear path. */
    double tm = INFINITY;
    int32_t j = 0, depth = 0;
    for (;;) {
      const double* l = target + ((size_t)b * (size_t)nn + (size_t)j) * (size_t)V;
      orc_softmax(l, V, T, p, NULL, NULL);
      double pz = 1.0;
      int moved = 0;
      if (irow[j] >= 0) {
        const int32_t* X = node_draft_tokens + ((size_t)b * (size_t)I + (size_t)irow[j]) * (size_t)N;
        double sigma, c[8], w[8], gap;
        for (int n = 0; n < N; ++n) {
          const double* d = draft + (((size_t)b * (size_t)I + (size_t)irow[j]) * (size_t)N + (size_t)n) * (size_t)V;
          orc_draft_dist(d, V, draft_kind, T, qn + (size_t)n * (size_t)V, &sigma);
          c[n] = qn[(size_t)n * (size_t)V + (size_t)X[n]];
        }
        orc_fusion_weights(N, c, weight_mode, w, &gap);
        if (weight_mode == ORC_W_WINNER) tm = dmin(tm, gap); /* the only argmax in a tree */
        for (int64_t v = 0; v < V; ++v) {
          double s = 0.0;
          for (int n = 0; n < N; ++n) s += w[n] * qn[(size_t)n * (size_t)V + (size_t)v];
          q[v] = s;
        }
        for (int32_t ch = j + 1; ch < nn; ++ch) {
          if (par[ch] != j) continue;
          const int32_t x = tok[ch];
          double u = orc_uniform(seed, rid, (uint32_t)ch, step, ORC_TAG_ACCEPT);
          double px = p[x] / pz;
          tm = dmin(tm, fabs(u - px / q[x]));
          if (u * q[x] < px) { /* accept: move to the child */
            an[depth] = ch;
            out[depth] = x;
            depth++;
            j = ch;
            moved = 1;
            break;
          }
          /* reject: p <- norm(max(0, p - q)); q <- q without x, renormalised */
          double Z = 0.0;
          for (int64_t v = 0; v < V; ++v) {
            double d = p[v] / pz - q[v];
            r[v] = d > 0.0 ? d : 0.0;
            Z += r[v];
          }
          if (Z == 0.0) {
            status[b] |= ORC_INFO_DEGENERATE_RESIDUAL; /* keep p (reading #11) */
          } else {
            memcpy(p, r, sizeof(double) * (size_t)V);
            pz = Z;
          }
          double qx = q[x];
          q[x] = 0.0;
          if (qx < 1.0)
            for (int64_t v = 0; v < V; ++v) q[v] /= (1.0 - qx);
        }
      }
      if (moved) continue;
      /* children exhausted, or a leaf: y ~ p with U(rid, j, SAMPLE) */
      double us = orc_uniform(seed, rid, (uint32_t)j, step, ORC_TAG_SAMPLE), ms;
      int64_t y = orc_invcdf(p, V, us, &ms);
      tm = dmin(tm, ms);
      out[depth] = (int32_t)y;
      accept_len[b] = depth;
      break;
    }
    if (tie_margin) tie_margin[b] = tm;
  }
  free(p); free(q); free(r); free(qn);
  return 0;
}

/* Drafter-side Fuse of one iteration (NEXT-2): Alg. 1 Fuse and Eq. 4's first line
 * over the drafters' greedy tokens, written out step by step. */
int orc_fuse_step(int32_t B, int32_t N, int64_t V, const double* logits, double temperature,
                  int32_t* own_tokens, double* conf, int32_t* fused_token, int32_t* winner,
                  int32_t* status, double* conf_gap) {
  if (B < 0 || N < 1 || V < 1 || !(temperature > 0.0) || !logits) return 1;
  for (int32_t b = 0; b < B; ++b) {
    int st = 0;
    double c[64];
    int64_t X[64];
    if (N > 64) return 1;
    for (int32_t n = 0; n < N && !st; ++n) {
      const double* l = logits + ((int64_t)b * N + n) * V;
      int64_t am = -1;
      st = orc_argmax(l, V, &am); /* X_n: the drafter's own (greedy) token */
      if (st) break;
      double M = 0.0, S = 0.0;
      double* p = (double*)malloc(sizeof(double) * (size_t)V);
      if (!p) return 1;
      st = orc_softmax(l, V, temperature, p, &M, &S);
      if (!st) c[n] = p[am]; /* c_n = P(X_n) */
      free(p);
      X[n] = am;
    }
    status[b] = st;
    if (st) {
      for (int32_t n = 0; n < N; ++n) { own_tokens[(int64_t)b * N + n] = -1; conf[(int64_t)b * N + n] = NAN; }
      fused_token[b] = -1;
      winner[b] = -1;
      if (conf_gap) conf_gap[b] = NAN;
      continue;
    }
    int nstar = 0; /* Eq. 4: the most confident drafter, lowest n on ties */
    for (int32_t n = 1; n < N; ++n)
      if (c[n] > c[nstar]) nstar = n;
    double second = -1.0;
    for (int32_t n = 0; n < N; ++n)
      if (n != nstar && c[n] > second) second = c[n];
    for (int32_t n = 0; n < N; ++n) {
      own_tokens[(int64_t)b * N + n] = (int32_t)X[n];
      conf[(int64_t)b * N + n] = c[n];
    }
    fused_token[b] = (int32_t)X[nstar];
    winner[b] = nstar;
    if (conf_gap) conf_gap[b] = (N > 1) ? (c[nstar] - second) / c[nstar] : INFINITY;
  }
  return 0;
}

/* Routing feedback (NEXT-3): Eq. 1 then Eq. 2, written out. */
static double orc_cos(const double* a, const double* b, int64_t H) {
  double ab = 0.0, aa = 0.0, bb = 0.0;
  for (int64_t h = 0; h < H; ++h) { ab += a[h] * b[h]; aa += a[h] * a[h]; bb += b[h] * b[h]; }
  if (aa == 0.0 || bb == 0.0) return 0.0;
  return ab / (sqrt(aa) * sqrt(bb));
}

int orc_route_update(int32_t B, int32_t N, int32_t K, int64_t V, int64_t Hd, const int32_t* draft_tokens,
                     const double* conf, const int32_t* accepted, int64_t acc_stride, const int32_t* accept_len,
                     const double* emb, const uint8_t* participating, double decay, double eps, double* M,
                     double* d_out, int32_t* status) {
  if (B < 0 || N < 1 || K < 1 || V < 1 || Hd < 1 || acc_stride < K || !(eps > 0.0 && eps < 0.5)) return 1;
  for (int32_t b = 0; b < B; ++b) {
    status[b] = 0;
    const int32_t L = accept_len[b];
    if (L < 0) continue; /* a request whose verification failed: no feedback */
    int bad = 0;
    for (int32_t n = 0; n < N; ++n)
      for (int32_t i = 0; i < K; ++i) {
        const int32_t x = draft_tokens[((int64_t)b * N + n) * K + i];
        if (x < 0 || x >= V) bad = 1;
      }
    for (int32_t i = 0; i < K && i < L; ++i) {
      const int32_t a = accepted[(int64_t)b * acc_stride + i];
      if (a < 0 || a >= V) bad = 1;
    }
    if (bad) { status[b] = 2; continue; }
    for (int32_t n = 0; n < N; ++n) {
      const int64_t bn = (int64_t)b * N + n;
      if (participating && !participating[bn]) {
        M[bn] = 0.5 + decay * (M[bn] - 0.5); /* non-participating entries decay to 0.5 */
        continue;
      }
      double m = 0.0;
      for (int32_t i = 0; i < K; ++i) {
        double d = 0.0;
        if (i < L) { /* Eq. 1 */
          const int32_t a = accepted[(int64_t)b * acc_stride + i];
          const int32_t x = draft_tokens[bn * K + i];
          d = orc_cos(emb + (int64_t)a * Hd, emb + (int64_t)x * Hd, Hd);
        }
        if (d_out) d_out[bn * K + i] = d;
        double c = conf[bn * K + i];
        c = c < eps ? eps : (c > 1.0 - eps ? 1.0 - eps : c);
        d = d < eps ? eps : (d > 1.0 - eps ? 1.0 - eps : d);
        m += c * d / (c * d + (1.0 - c) * (1.0 - d)); /* Eq. 2 */
      }
      M[bn] = m / K;
    }
  }
  return 0;
}

/* TreeSelection (NEXT-4, reading #25), step by step: trie insertion, node scores, top-budget
 * pruning, breadth-first renumbering. */
int orc_tree_select(int32_t B, int32_t S, int32_t K, const int32_t* tokens, const double* conf, int32_t budget,
                    int32_t* n_nodes, int32_t* parent, int32_t* token, double* score, int32_t* depth) {
  if (B < 0 || S < 1 || K < 1 || budget < 0 || S * K > 4096) return 1;
  const int cap = S * K + 1;
  int32_t* tp = (int32_t*)malloc(sizeof(int32_t) * cap); /* trie: parent, token, depth, score */
  int32_t* tt = (int32_t*)malloc(sizeof(int32_t) * cap);
  int32_t* td = (int32_t*)malloc(sizeof(int32_t) * cap);
  double* ts = (double*)malloc(sizeof(double) * cap);
  int32_t* keep = (int32_t*)malloc(sizeof(int32_t) * cap);
  int32_t* newid = (int32_t*)malloc(sizeof(int32_t) * cap);
  if (!tp || !tt || !td || !ts || !keep || !newid) return 1;
  for (int32_t b = 0; b < B; ++b) {
    int n = 1;
    tp[0] = -1; tt[0] = -1; td[0] = 0; ts[0] = 1.0;
    for (int32_t s2 = 0; s2 < S; ++s2) { /* 1. merge the branches into a prefix tree */
      int cur = 0;
      double prod = 1.0;
      for (int32_t i = 0; i < K; ++i) {
        const int32_t x = tokens[((int64_t)b * S + s2) * K + i];
        if (x < 0) break;
        prod *= conf[((int64_t)b * S + s2) * K + i];
        int child = -1;
        for (int c = 1; c < n; ++c)
          if (tp[c] == cur && tt[c] == x) { child = c; break; }
        if (child < 0) { child = n++; tp[child] = cur; tt[child] = x; td[child] = td[cur] + 1; ts[child] = prod; }
        else if (prod > ts[child]) ts[child] = prod; /* 2. the best branch product reaching it */
        cur = child;
      }
    }
    /* 3. keep the budget best non-root nodes: score desc, depth asc, creation order */
    for (int c = 0; c < n; ++c) keep[c] = (c == 0);
    const int nk = (n - 1 < budget) ? n - 1 : budget;
    for (int r = 0; r < nk; ++r) {
      int best = -1;
      for (int c = 1; c < n; ++c) {
        if (keep[c]) continue;
        if (best < 0 || ts[c] > ts[best] || (ts[c] == ts[best] && (td[c] < td[best] || (td[c] == td[best] && c < best))))
          best = c;
      }
      keep[best] = 1;
    }
    /* 4. breadth-first renumbering; siblings by (score desc, creation) */
    for (int c = 0; c < n; ++c) newid[c] = -1;
    newid[0] = 0;
    int next = 1;
    for (int d = 1; d <= K; ++d) {
      for (int p = 0; p < next; ++p) { /* parents in their new order */
        int old_p = -1;
        for (int c = 0; c < n; ++c)
          if (newid[c] == p) { old_p = c; break; }
        for (;;) { /* the best remaining kept child of old_p at depth d */
          int best = -1;
          for (int c = 1; c < n; ++c) {
            if (!keep[c] || newid[c] >= 0 || tp[c] != old_p || td[c] != d) continue;
            if (best < 0 || ts[c] > ts[best] || (ts[c] == ts[best] && c < best)) best = c;
          }
          if (best < 0) break;
          newid[best] = next++;
        }
      }
    }
    const int64_t o = (int64_t)b * (budget + 1);
    for (int j = 0; j <= budget; ++j) { parent[o + j] = -1; token[o + j] = -1; score[o + j] = 0.0; depth[o + j] = -1; }
    for (int c = 0; c < n; ++c) {
      if (!keep[c]) continue;
      const int j = newid[c];
      parent[o + j] = (c == 0) ? -1 : newid[tp[c]];
      token[o + j] = tt[c];
      score[o + j] = ts[c];
      depth[o + j] = td[c];
    }
    n_nodes[b] = next;
  }
  free(tp); free(tt); free(td); free(ts); free(keep); free(newid);
  return 0;
}
