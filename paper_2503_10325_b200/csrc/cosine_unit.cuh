// cosine_unit.cuh — legacy one-cluster-per-unit kernel (fuse_drafts / sample_residual /
// SAMPLE select); being retired.
#pragma once

#include <cooperative_groups.h>
#include "cosine_common.cuh"

namespace cosine {
namespace cg = cooperative_groups;

enum Mode : int { kModeVerify = 0, kModeFuse = 1, kModeSample = 2 };

struct UnitRec {  // one per (request, position); 32 bytes
  int32_t xstar;
  int32_t y;
  int32_t flags;  // bit0 accept, bit1 y valid, bit2 degenerate, bits 8..15 status
  float m_fa;     // min(fusion gap, acceptance margin)
  float m_s;      // sampling margin
  float z;        // residual mass (probability units)
  float pad0, pad1;
};

struct Params {
  int mode;
  int B, k, N;
  int64_t V;  // vocabulary width of this context
  int64_t ld_t, ld_q, ld_fq;
  int64_t ngroups, gfull, gpc;  // groups, full groups, groups per CTA
  int C;
  float T, k2f;
  double k2d;
  int greedy, weight_mode, select_mode;
  const void* target;
  const void* draft;
  const int32_t* draft_tokens;
  const int32_t* draft_len;
  const uint64_t* rids;
  uint64_t seed;
  uint32_t step;
  int32_t* accept_len;
  int32_t* out_tokens;
  int32_t* status;
  cosine_debug_t dbg;
  int32_t* fused_tokens;
  float* w_out;
  float* norm_out;
  float* fused_q;
  const float* row_max;
  const float* row_sumexp;
  const float* w_in;
  const float* norm_in;
  const uint32_t* node_ids;
  int32_t* out_token;
  UnitRec* recs;
  int32_t* done;
  int32_t* first_rej;
};

struct CtaRec {
  float tmax;    // T > 0: max logit of the chunk; greedy: best value
  int32_t bad;   // bit0 target non-finite (greedy), bit1 negative drafter prob
  int64_t targ;  // greedy argmax (global index), -1 if none
  double tsum;   // sum exp2((l - tmax) k2) over the chunk
  float dmax[kMaxN];
  double dsum[kMaxN];
};


struct SampleOut {
  int64_t y;
  float margin, z;
  int32_t degenerate;
  float tx;
  float dx[kMaxN];
};

struct UnitState {  // CTA 0, thread 0 only
  int32_t status, nstar, xstar, accept, y, sampled, degenerate, last_kind;
  double M, S, px, qx, u;
  int64_t amax;
  float Mf, m_fa, m_s, z;
  double sig[kMaxN], c[kMaxN], w[kMaxN];
  float dmax[kMaxN];
};


template <typename TT, typename TQ, bool kLogits, int NMAX>
__global__ void __launch_bounds__(kThreads, (NMAX <= 4 ? 4 : 2)) unit_kernel(const Params P) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = P.C;
  const int rank = (int)cluster.block_rank();
  const int64_t unit = blockIdx.x / C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  __shared__ CtaRec s_rec[kMaxC];
  __shared__ Decision s_dec[2];
  __shared__ double s_z[2][kMaxC];
  __shared__ SampleOut s_out;
  __shared__ UnitState s_st;
  __shared__ float s_gx[kMaxN + 1][kMaxN];  // [m][n]: drafter m (m == N: target) at X_n
  __shared__ int32_t s_tok[kMaxN];
  __shared__ float s_wf[kWarps][1 + kMaxN];
  __shared__ float s_wv[kWarps];
  __shared__ int64_t s_wi[kWarps];
  __shared__ double s_wd[kWarps][1 + kMaxN];
  __shared__ int32_t s_wbad[kWarps];
  __shared__ double s_scan[kWarps];
  __shared__ int64_t s_found;
  __shared__ float s_margin;
  __shared__ double s_seg[kMaxSeg];

  // ---------------- unit decode ----------------
  int b = 0, i = 0, g = 0;
  bool has_t = false, has_d = false;
  const TT* trow = nullptr;
  const TQ* drow = nullptr;
  const int N = P.N;
  if (P.mode == kModeVerify) {
    // position-major order: when position i of a request runs, its earlier positions have
    // (mostly) decided, so the first-rejection gate below is nearly exact
    i = (int)(unit / P.B);
    b = (int)(unit % P.B);
    g = P.draft_len ? P.draft_len[b] : P.k;
    if (g < 1 || g > P.k) {  // per-request error, no unit of b runs
      if (i == 0 && rank == 0 && tid == 0) {
        P.accept_len[b] = -1;
        for (int j = 0; j <= P.k; ++j) P.out_tokens[(int64_t)b * (P.k + 1) + j] = -1;
        P.status[b] = COSINE_REQ_BAD_DRAFT_LEN;
      }
      return;
    }
    if (i > g) return;  // rows past gamma_b are never read
    has_t = true;
    has_d = (i < g);
    trow = (const TT*)P.target + ((int64_t)b * (P.k + 1) + i) * P.ld_t;
    if (has_d) drow = (const TQ*)P.draft + ((int64_t)b * P.k + i) * N * P.ld_q;
  } else if (P.mode == kModeFuse) {
    i = (int)(unit / P.B);
    b = (int)(unit % P.B);
    g = P.k;
    has_d = true;
    drow = (const TQ*)P.draft + ((int64_t)b * P.k + i) * N * P.ld_q;
  } else {
    b = (int)unit;
    has_t = true;
    has_d = (P.draft != nullptr);
    trow = (const TT*)P.target + (int64_t)b * P.ld_t;
    if (has_d) drow = (const TQ*)P.draft + (int64_t)b * N * P.ld_q;
  }
  const int Nd = has_d ? N : 0;
  const uint64_t rid = P.rids[b];
  // solo: the C-1 helper CTAs leave as soon as their statistics are in CTA 0; CTA 0 alone
  // decides and (rarely: first rejection / bonus) samples from the L2-resident rows.
  // Cooperative (all CTAs stay) only when every unit needs a full-row pass after the stats:
  // x* ~ q (SAMPLE select) or materialising q (fuse_drafts with fused_q).
  const bool solo = !(P.select_mode == COSINE_SEL_SAMPLE || (P.mode == kModeFuse && P.fused_q));
  __shared__ __align__(8) uint64_t s_bar;
  if (solo) {
    if (rank == 0 && tid == 0) {
      mbar_init(&s_bar, (uint32_t)C);
      fence_mbar_init_cluster();
    }
    cluster_arrive_relaxed();
  }

  // ---------------- candidate gathers (CTA 0; in flight during the stream) ----------------
  const int n_gath = (P.mode != kModeSample && has_d) ? N * (N + (has_t ? 1 : 0)) : 0;
  const bool gact = (rank == 0 && tid < n_gath);
  int32_t gtok = -1;
  float gval = 0.f;
  if (gact) {
    const int n = tid % N, m = tid / N;
    gtok = P.draft_tokens[((int64_t)b * P.k + i) * N + n];
    if (gtok >= 0 && (int64_t)gtok < P.V)
      gval = (m < N) ? load_one(drow + (int64_t)m * P.ld_q, gtok) : load_one(trow, gtok);
  }

  // ---------------- pass 1: stream the chunk once ----------------
  const float k2 = P.k2f;
  float tm = kNegBig, ts = 0.f;          // online max / sum-exp (T > 0)
  float tb = -INFINITY;                  // greedy best
  int64_t ti = -1;
  bool tbad = false;
  float dm[NMAX], ds[NMAX];
#pragma unroll
  for (int n = 0; n < NMAX; ++n) { dm[n] = kNegBig; ds[n] = 0.f; }
  bool dneg = false;
  const bool greedy = P.greedy != 0;
  const int64_t gb = (int64_t)rank * P.gpc;
  const int64_t ge = min(P.ngroups, gb + P.gpc);

  auto target_step = [&](const float (&f)[8], int64_t gi) {
    if (greedy) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (f[e] > tb) { tb = f[e]; ti = gi * kGroup + e; }
        tbad |= !(f[e] <= 3.402823466e+38f);
      }
    } else {
      const float gm = max8(f);
      if (gm > tm) { ts *= ex2((tm - gm) * k2); tm = gm; }
      float e8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) e8[e] = ex2((f[e] - tm) * k2);
      ts += sum8(e8);
    }
  };
  auto draft_step = [&](int n, const float (&f)[8]) {
    if (kLogits) {
      const float gm = max8(f);
      if (gm > dm[n]) { ds[n] *= ex2((dm[n] - gm) * k2); dm[n] = gm; }
      float e8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) e8[e] = ex2((f[e] - dm[n]) * k2);
      ds[n] += sum8(e8);
    } else {
      ds[n] += sum8(f);
    }
  };

  for (int64_t gi = gb + tid; gi < ge; gi += kThreads) {
    float f[8];
    if (gi < P.gfull) {
      Group<TT> tv;
      Group<TQ> dv[NMAX];
      if (has_t) tv.load(trow, gi);
#pragma unroll
      for (int n = 0; n < NMAX; ++n)
        if (n < Nd) dv[n].load(drow + (int64_t)n * P.ld_q, gi);
      if (has_t) { tv.unpack(f); target_step(f, gi); }
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n < Nd) {
          dv[n].unpack(f);
          if (!kLogits && dv[n].any_sign()) {
#pragma unroll
            for (int e = 0; e < 8; ++e) dneg |= (f[e] < 0.f);
          }
          draft_step(n, f);
        }
      }
    } else {
      if (has_t) { load_partial(trow, gi, P.V, -INFINITY, f); target_step(f, gi); }
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n < Nd) {
          load_partial(drow + (int64_t)n * P.ld_q, gi, P.V, kLogits ? -INFINITY : 0.f, f);
          if (!kLogits) {
#pragma unroll
            for (int e = 0; e < 8; ++e) dneg |= (f[e] < 0.f);
          }
          draft_step(n, f);
        }
      }
    }
  }
  if (gact) s_gx[tid / N][tid % N] = gval;
  if (rank == 0 && tid < N && n_gath > 0) s_tok[tid] = gtok;

  // ---------------- CTA reduction -> record pushed to CTA 0 over DSMEM ----------------
  {
    float tmw = kNegBig;
    float tbw = tb;
    int64_t tiw = ti;
    if (has_t) {
      if (greedy) warp_argmax(tbw, tiw);
      else tmw = warp_max(tm);
    }
    float dmw[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) dmw[n] = (kLogits && n < Nd) ? warp_max(dm[n]) : kNegBig;
    if (lane == 0) {
      s_wf[warp][0] = tmw;
      s_wv[warp] = tbw;
      s_wi[warp] = tiw;
#pragma unroll
      for (int n = 0; n < NMAX; ++n) s_wf[warp][1 + n] = dmw[n];
    }
    __syncthreads();
    float Mc = kNegBig;
    float dMc[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) dMc[n] = kNegBig;
    for (int w = 0; w < kWarps; ++w) {
      Mc = fmaxf(Mc, s_wf[w][0]);
#pragma unroll
      for (int n = 0; n < NMAX; ++n) dMc[n] = fmaxf(dMc[n], s_wf[w][1 + n]);
    }
    // sums rescaled to the CTA max, in fp64 (exp2 of an exact fp64 difference)
    double tsd = 0.0;
    if (has_t && !greedy && ts != 0.f) tsd = (double)ts * exp2(((double)tm - (double)Mc) * P.k2d);
    double dsd[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      dsd[n] = 0.0;
      if (n < Nd) {
        if (kLogits) {
          if (ds[n] != 0.f) dsd[n] = (double)ds[n] * exp2(((double)dm[n] - (double)dMc[n]) * P.k2d);
        } else {
          dsd[n] = (double)ds[n];
        }
      }
    }
    tsd = warp_sum(tsd);
#pragma unroll
    for (int n = 0; n < NMAX; ++n) dsd[n] = warp_sum(dsd[n]);
    const int bad = (__any_sync(0xffffffffu, tbad) ? 1 : 0) | (__any_sync(0xffffffffu, dneg) ? 2 : 0);
    if (lane == 0) {
      s_wd[warp][0] = tsd;
#pragma unroll
      for (int n = 0; n < NMAX; ++n) s_wd[warp][1 + n] = dsd[n];
      s_wbad[warp] = bad;
    }
    __syncthreads();
    if (tid == 0) {
      CtaRec rec;
      rec.tmax = Mc;
      rec.targ = -1;
      rec.bad = 0;
      rec.tsum = 0.0;
      if (greedy) {
        float bv = -INFINITY;
        int64_t bi = -1;
        for (int w = 0; w < kWarps; ++w) {
          const float v = s_wv[w];
          const int64_t ix = s_wi[w];
          if (ix >= 0 && (bi < 0 || v > bv || (v == bv && ix < bi))) { bv = v; bi = ix; }
        }
        rec.tmax = bv;
        rec.targ = bi;
      }
      for (int w = 0; w < kWarps; ++w) {
        rec.tsum += s_wd[w][0];
        rec.bad |= s_wbad[w];
      }
#pragma unroll
      for (int n = 0; n < kMaxN; ++n) {
        rec.dmax[n] = kNegBig;
        rec.dsum[n] = 0.0;
      }
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        rec.dmax[n] = dMc[n];
        double sacc = 0.0;
        for (int w = 0; w < kWarps; ++w) sacc += s_wd[w][1 + n];
        rec.dsum[n] = sacc;
      }
      if (solo) cluster_wait();  // CTA 0's mbarrier is initialised
      CtaRec* dst = cluster.map_shared_rank(s_rec, 0) + rank;
      *dst = rec;
      if (solo) mbar_remote_arrive(&s_bar, 0);
    }
  }
  if (solo) {
    if (tid != 0) cluster_wait();
    if (rank != 0) return;  // helpers leave: no DSMEM access to them from now on
    if (tid == 0) mbar_wait_parity(&s_bar, 0);
    __syncthreads();
  } else {
    cluster.sync();
  }
  const int bcast = solo ? 1 : C;

  // ---------------- decision loop ----------------
  for (int round = 0;; ++round) {
    if (rank == 0 && tid == 0) {
      UnitState& st = s_st;
      Decision d;
      d.need = 0;
      d.kind = kWBonus;
      d.xstar = -1;
      d.node = 0;
      d.u = 0.0;
      d.k2 = k2;
      d.M = 0.f;
      d.invS = 0.f;
      for (int n = 0; n < kMaxN; ++n) { d.a[n] = 0.f; d.dm[n] = 0.f; }
      bool want_accept = false;
      if (round == 0) {
        // combine the C records in rank order (= ascending vocabulary chunks)
        st.status = 0;
        st.accept = 1;
        st.y = -1;
        st.sampled = 0;
        st.degenerate = 0;
        st.xstar = -1;
        st.nstar = 0;
        st.m_fa = INFINITY;
        st.m_s = INFINITY;
        st.z = NAN;
        st.px = st.qx = st.u = NAN;
        st.M = 0.0;
        st.S = 0.0;
        st.amax = -1;
        st.last_kind = -1;
        bool t_nf = false, t_empty = false, d_nf = false, d_empty = false, tok_bad = false,
             zero = false;
        if (has_t) {
          if (greedy) {
            float bv = -INFINITY;
            int64_t bi = -1;
            int bad = 0;
            for (int r = 0; r < C; ++r) {
              const CtaRec& rc = s_rec[r];
              bad |= rc.bad;
              if (rc.targ >= 0 && (bi < 0 || rc.tmax > bv)) { bv = rc.tmax; bi = rc.targ; }
            }
            t_nf = (bad & 1) != 0;
            t_empty = (bi < 0);
            st.amax = bi;
            st.Mf = bv;
            st.M = bv;
          } else {
            float M = kNegBig;
            for (int r = 0; r < C; ++r) M = fmaxf(M, s_rec[r].tmax);
            double S = 0.0;
            for (int r = 0; r < C; ++r) {
              const double sr = s_rec[r].tsum;
              if (sr != 0.0) S += sr * exp2(((double)s_rec[r].tmax - (double)M) * P.k2d);
            }
            st.Mf = M;
            st.M = M;
            st.S = S;
            t_nf = !isfinite(S) || !isfinite(M);
            t_empty = !t_nf && !(S > 0.0);
          }
        }
        if (has_d) {
          int bad = 0;
          for (int r = 0; r < C; ++r) bad |= s_rec[r].bad;
          if (bad & 2) d_nf = true;
          for (int n = 0; n < N; ++n) {
            double s = 0.0;
            float mx = kNegBig;
            if (kLogits) {
              for (int r = 0; r < C; ++r) mx = fmaxf(mx, s_rec[r].dmax[n]);
              for (int r = 0; r < C; ++r) {
                const double sr = s_rec[r].dsum[n];
                if (sr != 0.0) s += sr * exp2(((double)s_rec[r].dmax[n] - (double)mx) * P.k2d);
              }
              if (!isfinite(mx)) d_nf = true;
            } else {
              for (int r = 0; r < C; ++r) s += s_rec[r].dsum[n];
            }
            st.sig[n] = s;
            st.dmax[n] = mx;
            if (!isfinite(s)) d_nf = true;
            else if (!(s > 0.0)) d_empty = true;
          }
          if (P.mode != kModeSample)
            for (int n = 0; n < N; ++n)
              if (s_tok[n] < 0 || (int64_t)s_tok[n] >= P.V) tok_bad = true;
        }
        if (P.mode == kModeSample) {
          d_empty = false;  // the caller's sigma is used (cosine_sample_residual)
          if (P.row_max) t_empty = false;
        }
        int stc = 0;
        if (tok_bad) stc = COSINE_REQ_TOKEN_OUT_OF_RANGE;
        else if (t_nf || d_nf) stc = COSINE_REQ_NONFINITE_INPUT;
        else if (t_empty || d_empty) stc = COSINE_REQ_EMPTY_ROW;
        if (!stc && has_d && P.mode != kModeSample) {
          // confidences c_n = q_n(X_n) and Eq. 4 fusion (ties -> lowest n)
          for (int n = 0; n < N; ++n) {
            const double dv = (double)s_gx[n][n];
            st.c[n] = kLogits ? exp2((dv - (double)st.dmax[n]) * P.k2d) / st.sig[n] : dv / st.sig[n];
            if (st.c[n] == 0.0) zero = true;
          }
          if (zero) stc = COSINE_REQ_ZERO_PROB_DRAFT;
        }
        st.status = stc;
        if (!stc && has_d && P.mode != kModeSample) {
          int ns = 0;
          for (int n = 1; n < N; ++n)
            if (st.c[n] > st.c[ns]) ns = n;
          double second = -1.0;
          for (int n = 0; n < N; ++n)
            if (n != ns && st.c[n] > second) second = st.c[n];
          const float gap = (N > 1) ? (float)((st.c[ns] - second) / st.c[ns]) : INFINITY;
          st.nstar = ns;
          if (P.weight_mode == COSINE_W_CONF) {
            double sc = 0.0;
            for (int n = 0; n < N; ++n) sc += st.c[n];
            for (int n = 0; n < N; ++n) st.w[n] = st.c[n] / sc;
          } else if (P.weight_mode == COSINE_W_UNIFORM) {
            for (int n = 0; n < N; ++n) st.w[n] = 1.0 / (double)N;
          } else {
            for (int n = 0; n < N; ++n) st.w[n] = (n == ns) ? 1.0 : 0.0;
          }
          if (P.select_mode == COSINE_SEL_ARGMAX) {
            st.m_fa = gap;
            st.xstar = s_tok[ns];
            // gathered o(x*) and q(x*)
            if (P.weight_mode == COSINE_W_POINT) {
              st.qx = 1.0;
            } else {
              double q = 0.0;
              for (int m = 0; m < N; ++m) {
                const double dv = (double)s_gx[m][ns];
                const double qm = kLogits ? exp2((dv - (double)st.dmax[m]) * P.k2d) / st.sig[m]
                                          : dv / st.sig[m];
                q += st.w[m] * qm;
              }
              st.qx = q;
            }
            if (has_t && !greedy) st.px = exp2(((double)s_gx[N][ns] - st.M) * P.k2d) / st.S;
            want_accept = (P.mode == kModeVerify);
          } else {
            // SAMPLE select: x* ~ q with U(rid, i+1, FUSE)
            d.need = 1;
            d.kind = kWFuseQ;
            d.node = (uint32_t)(i + 1);
            d.u = philox_u24(P.seed, rid, (uint32_t)(i + 1), P.step, kTagFuse);
          }
        }
        if (!stc && P.mode == kModeVerify && !has_d) {  // bonus row (i == gamma_b)
          if (greedy) {
            st.y = (int)st.amax;
          } else if (*((volatile int32_t*)&P.first_rej[b]) >= g) {
            d.need = 1;
            d.kind = kWBonus;
            d.node = (uint32_t)g;
            d.u = philox_u24(P.seed, rid, (uint32_t)g, P.step, kTagSample);
          }
        }
        if (!stc && P.mode == kModeSample) {
          if (greedy) {
            st.y = (int)st.amax;
          } else {
            if (P.row_max) {
              st.M = (double)P.row_max[b];
              st.Mf = P.row_max[b];
              st.S = (double)P.row_sumexp[b];
              if (!(st.S > 0.0) || !isfinite(st.S) || !isfinite(st.M)) stc = COSINE_REQ_EMPTY_ROW;
            }
            if (has_d)
              for (int n = 0; n < N; ++n) {
                const float nv = P.norm_in[(int64_t)b * N + n];
                if (!(nv > 0.f) || !isfinite(nv)) stc = COSINE_REQ_EMPTY_ROW;
                st.w[n] = (double)P.w_in[(int64_t)b * N + n];
                st.sig[n] = (double)nv;
              }
            st.status = stc;
            if (!stc) {
              d.need = 1;
              d.kind = has_d ? kWResidual : kWBonus;
              d.node = P.node_ids[b];
              d.u = philox_u24(P.seed, rid, d.node, P.step, kTagSample);
            }
          }
        }
      } else {
        // result of the previous sampling round (in s_out)
        const int lk = st.last_kind;
        if (lk == kWFuseQ) {
          st.xstar = (int)s_out.y;
          st.m_fa = fmin_(st.m_fa, s_out.margin);
          if (st.xstar >= 0) {
            double q = 0.0;
            for (int m = 0; m < N; ++m) {
              const double dv = (double)s_out.dx[m];
              const double qm = kLogits ? exp2((dv - (double)st.dmax[m]) * P.k2d) / st.sig[m]
                                        : dv / st.sig[m];
              q += st.w[m] * qm;
            }
            st.qx = q;
            if (has_t && !greedy) st.px = exp2(((double)s_out.tx - st.M) * P.k2d) / st.S;
            want_accept = (P.mode == kModeVerify);
          }
        } else if (lk != kWWriteQ) {
          st.y = (int)s_out.y;
          st.sampled = 1;
          st.degenerate = s_out.degenerate;
          st.m_s = s_out.margin;
          st.z = s_out.z;
        }
      }
      if (want_accept) {
        // acceptance u * q(x*) < o(x*), i.e. u < min(1, o/q)
        st.u = philox_u24(P.seed, rid, (uint32_t)(i + 1), P.step, kTagAccept);
        if (greedy) {
          st.accept = ((int64_t)st.xstar == st.amax);
          st.y = (int)st.amax;
        } else {
          st.accept = (st.u * st.qx < st.px);
          st.m_fa = fmin_(st.m_fa, (float)fabs(st.u - st.px / st.qx));
          if (!st.accept) {
            const int old = atomicMin(&P.first_rej[b], i);
            if (old > i) {  // possibly the first rejection: resample
              d.need = 1;
              d.kind = (P.weight_mode == COSINE_W_POINT) ? kWPoint : kWResidual;
              d.node = (uint32_t)i;
              d.u = philox_u24(P.seed, rid, (uint32_t)i, P.step, kTagSample);
            }
          }
        }
      }
      if (!d.need && P.mode == kModeFuse && st.status == 0 && P.fused_q != nullptr &&
          st.last_kind != kWWriteQ && round <= 1) {
        d.need = 1;
        d.kind = kWWriteQ;
      }
      if (d.need) {
        d.M = st.Mf;
        d.invS = (float)(1.0 / st.S);
        d.xstar = st.xstar;
        for (int n = 0; n < N; ++n) {
          d.a[n] = (float)(st.w[n] / st.sig[n]);
          d.dm[n] = st.dmax[n];
        }
        st.last_kind = d.kind;
        s_out.y = -1;
        s_out.margin = 0.f;
        s_out.degenerate = 0;
        s_out.z = NAN;
      }
      if (solo) s_dec[round & 1] = d;
      else
        for (int r = 0; r < bcast; ++r) cluster.map_shared_rank(s_dec, r)[round & 1] = d;
    }
    if (solo) __syncthreads();
    else cluster.sync();
    const Decision d = s_dec[round & 1];
    if (!d.need) break;

    if (d.kind == kWWriteQ) {  // fuse_drafts: materialise q_i (or delta_{x*}) for this chunk
      float* qrow = P.fused_q + ((int64_t)b * P.k + i) * P.ld_fq;
      for (int64_t gi = gb + tid; gi < ge; gi += kThreads) {
        float w[8];
        if (P.weight_mode == COSINE_W_POINT) {
#pragma unroll
          for (int e = 0; e < 8; ++e) w[e] = (gi * kGroup + e == (int64_t)d.xstar) ? 1.f : 0.f;
        } else {
          group_weights<TT, TQ, kLogits, NMAX>(P, d, kWWriteQ, trow, drow, Nd, gi, w);
        }
        if (gi < P.gfull) {
          float4* o = reinterpret_cast<float4*>(qrow + gi * kGroup);
          o[0] = make_float4(w[0], w[1], w[2], w[3]);
          o[1] = make_float4(w[4], w[5], w[6], w[7]);
        } else {
          for (int e = 0; e < 8; ++e)
            if (gi * kGroup + e < P.V) qrow[gi * kGroup + e] = w[e];
        }
      }
      // no DSMEM traffic after this point: every CTA may leave
      if (rank == 0 && tid == 0) s_st.last_kind = kWWriteQ;
      break;
    }

    // ---- one inverse-CDF sampling round (reading #10) ----
    int kind = d.kind;
    int degenerate = 0;
    if (solo) {
      // CTA 0 alone over the whole row group: pass A = per-segment sums (one warp per
      // segment, no block barrier), then a tile scan of the crossing segment only.
      const int64_t segG = max((int64_t)kSegGroups, (P.ngroups + kMaxSeg - 1) / kMaxSeg);
      const int nseg = (int)((P.ngroups + segG - 1) / segG);
      for (int attempt = 0;; ++attempt) {
        __syncthreads();
        for (int sg = warp; sg < nseg; sg += kWarps) {
          double acc = 0.0;
          const int64_t e1 = min(P.ngroups, (sg + 1) * segG);
#pragma unroll 4
          for (int64_t gi = sg * segG + lane; gi < e1; gi += 32) {
            float w[8];
            group_weights<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, gi, w);
            acc += (double)sum8(w);
          }
          acc = warp_sum(acc);
          if (lane == 0) s_seg[sg] = acc;
        }
        __syncthreads();
        double Z = 0.0;
        for (int sg = 0; sg < nseg; ++sg) Z += s_seg[sg];
        if (!(Z > 0.0) && (kind == kWResidual || kind == kWPoint) && attempt == 0) {
          kind = kWProb;  // all mass cancelled: resample from o (reading #11)
          degenerate = 1;
          continue;
        }
        const double t = d.u * Z;
        int sstar = -1;
        double tc = 0.0, O = 0.0;
        for (int sg = 0; sg < nseg; ++sg) {
          const double z = s_seg[sg];
          if (O + z > t) { sstar = sg; tc = t - O; break; }
          O += z;
        }
        int64_t y = -1;
        float margin = 0.f;
        if (sstar >= 0)
          y = scan_range<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, sstar * segG,
                                                 min(P.ngroups, (sstar + 1) * segG), tc, Z, s_scan,
                                                 s_wi, &s_found, &s_margin);
        if (tid == 0) {
          margin = s_margin;
          s_out.y = y;
          s_out.margin = margin;
          s_out.degenerate = degenerate;
          s_out.z = (float)((kind == kWBonus) ? Z * (double)d.invS : Z);
          s_out.tx = 0.f;
          for (int n = 0; n < kMaxN; ++n) s_out.dx[n] = 0.f;
        }
        __syncthreads();
        break;
      }
      continue;
    }
    for (int attempt = 0;; ++attempt) {
      double acc = 0.0;
      for (int64_t gi = gb + tid; gi < ge; gi += kThreads) {
        float w[8];
        group_weights<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, gi, w);
        acc += (double)sum8(w);
      }
      const double zc = block_sum(acc, s_scan);
      if (tid == 0)
        for (int r = 0; r < C; ++r) cluster.map_shared_rank(&s_z[attempt & 1][0], r)[rank] = zc;
      cluster.sync();
      double Z = 0.0;
      for (int c = 0; c < C; ++c) Z += s_z[attempt & 1][c];
      if (!(Z > 0.0) && (kind == kWResidual || kind == kWPoint) && attempt == 0) {
        kind = kWProb;  // all mass cancelled: resample from o (reading #11)
        degenerate = 1;
        continue;
      }
      const double t = d.u * Z;
      int cstar = -1;
      double tc = 0.0, O = 0.0;
      for (int c = 0; c < C; ++c) {
        const double zcc = s_z[attempt & 1][c];
        if (O + zcc > t) { cstar = c; tc = t - O; break; }
        O += zcc;
      }
      if (rank == cstar) {
        const int64_t y = scan_range<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, gb, ge, tc, Z,
                                                             s_scan, s_wi, &s_found, &s_margin);
        (void)y;
        if (tid == 0) {
          SampleOut so;
          so.y = s_found;
          so.margin = s_margin;
          so.degenerate = degenerate;
          so.z = (float)((kind == kWBonus) ? Z * (double)d.invS : Z);
          so.tx = 0.f;
          for (int n = 0; n < kMaxN; ++n) so.dx[n] = 0.f;
          if (kind == kWFuseQ && so.y >= 0) {  // gathers at the sampled x*
            if (has_t) so.tx = load_one(trow, so.y);
            for (int n = 0; n < Nd; ++n) so.dx[n] = load_one(drow + (int64_t)n * P.ld_q, so.y);
          }
          *cluster.map_shared_rank(&s_out, 0) = so;
        }
      }
      cluster.sync();
      break;
    }
  }

  // ---------------- unit epilogue (CTA 0, thread 0) ----------------
  if (rank != 0 || tid != 0) return;
  UnitState& st = s_st;
  if (P.mode == kModeSample) {
    P.out_token[b] = st.status ? -1 : st.y;
    P.status[b] = st.status ? st.status
                            : ((st.degenerate ? COSINE_INFO_DEGENERATE_RESIDUAL : 0) |
                               (st.m_s < 1e-6f ? COSINE_INFO_NEAR_TIE : 0));
    return;
  }
  UnitRec rec;
  rec.xstar = st.xstar;
  rec.y = st.y;
  rec.flags = (st.accept ? 1 : 0) | ((st.y >= 0) ? 2 : 0) | (st.degenerate ? 4 : 0) | (st.status << 8);
  rec.m_fa = st.m_fa;
  rec.m_s = st.m_s;
  rec.z = st.z;
  rec.pad0 = rec.pad1 = 0.f;
  UnitRec* recs = P.recs + (int64_t)b * (P.k + 1);
  recs[i] = rec;

  if (P.mode == kModeFuse) {
    const int64_t o = (int64_t)b * P.k + i;
    P.fused_tokens[o] = st.status ? -1 : st.xstar;
    for (int n = 0; n < N; ++n) {
      if (P.w_out) P.w_out[o * N + n] = st.status ? NAN : (float)st.w[n];
      if (P.norm_out) P.norm_out[o * N + n] = st.status ? NAN : (float)st.sig[n];
    }
    __threadfence();
    const int old = atomicAdd(&P.done[b], 1);
    if (old == P.k - 1) {
      __threadfence();
      int err = 0;
      float tm = INFINITY;
      for (int j = 0; j < P.k; ++j) {
        const int f = __ldcg(&recs[j].flags);
        tm = fmin_(tm, fmin_(__ldcg(&recs[j].m_fa), __ldcg(&recs[j].m_s)));
        if (!err && ((f >> 8) & 0xff)) err = (f >> 8) & 0xff;
      }
      if (err)
        for (int j = 0; j < P.k; ++j) P.fused_tokens[(int64_t)b * P.k + j] = -1;
      P.status[b] = err ? err : (tm < 1e-6f ? COSINE_INFO_NEAR_TIE : 0);
      P.done[b] = 0;
    }
    return;
  }

  // verify: per-unit diagnostics
  {
    const cosine_debug_t& D = P.dbg;
    const int64_t ou = (int64_t)b * (P.k + 1) + i;
    if (D.row_max) D.row_max[ou] = st.Mf;
    if (D.row_sumexp) D.row_sumexp[ou] = greedy ? 0.f : (float)st.S;
    if (has_d) {
      const int64_t o = (int64_t)b * P.k + i;
      if (D.p_x) D.p_x[o] = (float)st.px;
      if (D.q_x) D.q_x[o] = (float)st.qx;
      if (D.accept_u) D.accept_u[o] = (float)st.u;
      if (D.fused_tokens) D.fused_tokens[o] = st.xstar;
      for (int n = 0; n < N; ++n) {
        if (D.draft_norm) D.draft_norm[o * N + n] = (float)st.sig[n];
        if (D.conf) D.conf[o * N + n] = (float)st.c[n];
        if (D.weights) D.weights[o * N + n] = (float)st.w[n];
      }
    }
  }
  __threadfence();
  const int old = atomicAdd(&P.done[b], 1);
  if (old != g) return;
  // last unit of request b: first rejection, emitted tokens
  __threadfence();
  int err = 0;
  for (int j = 0; j <= g; ++j) {
    const int f = __ldcg(&recs[j].flags);
    if ((f >> 8) & 0xff) { err = (f >> 8) & 0xff; break; }
  }
  int32_t* out = P.out_tokens + (int64_t)b * (P.k + 1);
  if (err) {
    P.accept_len[b] = -1;
    for (int j = 0; j <= P.k; ++j) out[j] = -1;
    P.status[b] = err;
  } else {
    int L = g;
    for (int j = 0; j < g; ++j)
      if (!(__ldcg(&recs[j].flags) & 1)) { L = j; break; }
    float tm = INFINITY;
    for (int j = 0; j < L; ++j) {
      out[j] = __ldcg(&recs[j].xstar);
      tm = fmin_(tm, __ldcg(&recs[j].m_fa));
    }
    if (L < g) tm = fmin_(tm, __ldcg(&recs[L].m_fa));
    tm = fmin_(tm, __ldcg(&recs[L].m_s));
    const int fL = __ldcg(&recs[L].flags);
    const int yL = __ldcg(&recs[L].y);
    out[L] = yL;
    for (int j = L + 1; j <= P.k; ++j) out[j] = -1;
    P.accept_len[b] = L;
    P.status[b] = ((fL & 4) ? COSINE_INFO_DEGENERATE_RESIDUAL : 0) |
                  (tm < 1e-6f ? COSINE_INFO_NEAR_TIE : 0) | ((fL & 2) ? 0 : 0xff);
    if (P.dbg.residual_mass) P.dbg.residual_mass[b] = __ldcg(&recs[L].z);
    if (P.dbg.tie_margin) P.dbg.tie_margin[b] = tm;
  }
  P.done[b] = 0;
  P.first_rej[b] = kNoReject;
}

}  // namespace cosine
