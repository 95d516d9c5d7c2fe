// cosine_verify.cu — sm_100a kernels + C ABI of libcosine_verify.so.
//
// One thread-block CLUSTER per "unit" = (request b, draft position i): the C CTAs of the
// cluster split the vocabulary into C contiguous chunks and stream, once, the unit's target
// logit row and its N drafter rows with 128-bit read-only loads (no tensor cores: nothing on
// this path is a contraction — it is HBM-bound).  Per-CTA statistics (online max / sum-exp,
// drafter sums, greedy argmax) are pushed into CTA 0's shared memory over DSMEM; CTA 0
// combines them in rank order, applies Eq. 4 fusion and the acceptance test
// u * q(x*) < p(x*), and — only for the first rejecting position of a request
// or for the bonus row — the whole cluster runs an inverse-CDF sampling
// round over the unit's rows, which are still L2-resident because they were streamed a few
// microseconds earlier.  The last unit of a request to finish (device-scope atomic counter)
// assembles accept_len / out_tokens.  Everything is one kernel launch per call.
//
// See DESIGN.md §5 for the roofline, byte accounting and the B200 design choices.

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "cosine_kernels.cuh"
#include "cosine_verify.h"

namespace cg = cooperative_groups;

namespace cosine {

enum Mode : int { kModeVerify = 0, kModeFuse = 1, kModeSample = 2 };
// Sampling weight kinds (what w(v) a sampling round draws from).
enum WKind : int {
  kWBonus = 0,     // exp((l - M)/T)
  kWResidual = 1,  // max(0, p - q), q = sum_n a_n d_n
  kWPoint = 2,     // max(0, p - delta_{x*})                    (POINT mode)
  kWFuseQ = 3,     // q (SAMPLE select: x* ~ q)                 (reading #3)
  kWProb = 4,      // p (degenerate residual fallback)    (reading #11)
  kWWriteQ = 5     // materialise q into fused_q (fuse_drafts)
};

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

struct Decision {
  int32_t need, kind, xstar;
  uint32_t node;
  double u;
  float M, invS, k2;
  float a[kMaxN], dm[kMaxN];
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

__device__ __forceinline__ float fmin_(float a, float b) { return a < b ? a : b; }

// Per-element sampling weights of one group (kinds above).
template <typename TT, typename TQ, bool kLogits, int NMAX, typename PP>
__device__ __forceinline__ void group_weights(const PP& P, const Decision& d, int kind,
                                              const TT* trow, const TQ* drow, int Nd, int64_t gi,
                                              float w[8]) {
  const bool need_t = (kind != kWFuseQ && kind != kWWriteQ);
  const bool need_q = (kind == kWResidual || kind == kWFuseQ || kind == kWWriteQ);
  float t[8], q[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) q[e] = 0.f;
  const bool full = gi < P.gfull;
  if (need_t) {
    if (full) {
      Group<TT> tv;
      tv.load(trow, gi);
      tv.unpack(t);
    } else {
      load_partial(trow, gi, P.V, -INFINITY, t);
    }
  }
  if (need_q) {
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      if (n < Nd) {
        float f[8];
        const TQ* row = drow + (int64_t)n * P.ld_q;
        if (full) {
          Group<TQ> dv;
          dv.load(row, gi);
          dv.unpack(f);
        } else {
          load_partial(row, gi, P.V, kLogits ? -INFINITY : 0.f, f);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float qv = kLogits ? ex2((f[e] - d.dm[n]) * d.k2) : f[e];
          q[e] = fmaf(d.a[n], qv, q[e]);
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    float x;
    if (kind == kWFuseQ || kind == kWWriteQ) {
      x = q[e];
    } else {
      const float pe = ex2((t[e] - d.M) * d.k2);
      if (kind == kWBonus) {
        x = pe;
      } else {
        const float p = pe * d.invS;
        if (kind == kWResidual) x = fmaxf(p - q[e], 0.f);
        else if (kind == kWPoint) x = (gi * kGroup + e == (int64_t)d.xstar) ? fmaxf(p - 1.f, 0.f) : p;
        else x = p;  // kWProb
      }
    }
    w[e] = (gi * kGroup + e < P.V) ? x : 0.f;
  }
}

// Block barrier: kBar == 0 -> __syncthreads; else named barrier 1 over kBar threads (the
// consumer warps of the persistent kernel, which must not wait for the producer warp).
template <int kBar>
__device__ __forceinline__ void sync_part() {
  if (kBar == 0) __syncthreads();
  else asm volatile("bar.sync 1, %0;" ::"r"(kBar) : "memory");
}

// Tile-ordered block scan of groups [sb, se): smallest v with C(v) > tc (C = running sum of
// w from sb), rounding fallback = last v with w(v) > 0 (reading #10).  Result valid in every
// thread; *s_margin (thread 0) = distance of tc to the chosen bin's edges / Z.
template <typename TT, typename TQ, bool kLogits, int NMAX, int kBar = 0, typename PP = Params>
__device__ __forceinline__ int64_t scan_range(const PP& P, const Decision& d, int kind,
                                           const TT* trow, const TQ* drow, int Nd, int64_t sb,
                                           int64_t se, double tc, double Z, double* s_scan,
                                           int64_t* s_wi, int64_t* s_found, float* s_margin) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;  // kBar: consumer-only barrier
  if (tid == 0) { *s_found = -1; *s_margin = 0.f; }
  sync_part<kBar>();
  double base = 0.0;
  for (int64_t t0 = sb; t0 < se; t0 += kThreads) {
    const int64_t gi = t0 + tid;
    float w[8];
    double s = 0.0;
    if (gi < se) {
      group_weights<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, gi, w);
      s = (double)sum8(w);
    }
    double incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double nb = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += nb;
    }
    if (lane == 31) s_scan[warp] = incl;
    sync_part<kBar>();
    double wpre = 0.0, tot = 0.0;
    for (int w2 = 0; w2 < kWarps; ++w2) {
      if (w2 < warp) wpre += s_scan[w2];
      tot += s_scan[w2];
    }
    const double excl = base + wpre + incl - s;
    if (gi < se && s > 0.0 && excl <= tc && tc < excl + s) {
      double cum = excl;
      int ef = -1;
      float mg = 0.f;
      for (int e = 0; e < 8; ++e) {
        const double prev = cum;
        cum += (double)w[e];
        if (cum > tc) {
          ef = e;
          mg = (float)(fmin(tc - prev, cum - tc) / Z);
          break;
        }
      }
      if (ef < 0) {
        for (int e = 7; e >= 0; --e)
          if (w[e] > 0.f) { ef = e; break; }
      }
      *s_found = gi * kGroup + ef;
      *s_margin = mg;
    }
    base += tot;
    sync_part<kBar>();
    if (*s_found >= 0) break;
  }
  if (*s_found < 0) {
    int64_t last = -1;
    for (int64_t gi = sb + tid; gi < se; gi += kThreads) {
      float w[8];
      group_weights<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, gi, w);
      for (int e = 0; e < 8; ++e)
        if (w[e] > 0.f) last = max(last, gi * kGroup + e);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    if (lane == 0) s_wi[warp] = last;
    sync_part<kBar>();
    if (tid == 0) {
      int64_t l2 = -1;
      for (int w2 = 0; w2 < kWarps; ++w2) l2 = max(l2, s_wi[w2]);
      *s_found = l2;
      *s_margin = 0.f;
    }
    sync_part<kBar>();
  }
  return *s_found;
}

// Block-wide sum of a double (result valid in thread 0).
__device__ __forceinline__ double block_sum(double x, double* s_buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  x = warp_sum(x);
  if (lane == 0) s_buf[warp] = x;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kWarps; ++w) r += s_buf[w];
  __syncthreads();
  return r;
}

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
#include "cosine_split.cuh"
#include "cosine_tree.cuh"
#include "cosine_shard.cuh"
#include "cosine_fuse_step.cuh"
#include "cosine_route.cuh"
#include "cosine_tree_select.cuh"
namespace cosine {

__global__ void init_scratch(int32_t* done, int32_t* first_rej, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) { done[j] = 0; first_rej[j] = kNoReject; }
}

using KernelFn = void (*)(Params);
using SplitFn = void (*)(SplitParams);
constexpr int kMaxChunks = 8;

template <typename TT, typename TQ>
void pick_split2(bool logits, int N, SplitFn* f) {
  if (logits) {
    f[0] = N <= 4 ? stats_kernel<TT, TQ, true, 4> : stats_kernel<TT, TQ, true, 8>;
    f[1] = decide_kernel<TT, TQ, true>;
    f[2] = N <= 4 ? resample_kernel<TT, TQ, true, 4> : resample_kernel<TT, TQ, true, 8>;
  } else {
    f[0] = N <= 4 ? stats_kernel<TT, TQ, false, 4> : stats_kernel<TT, TQ, false, 8>;
    f[1] = decide_kernel<TT, TQ, false>;
    f[2] = N <= 4 ? resample_kernel<TT, TQ, false, 4> : resample_kernel<TT, TQ, false, 8>;
  }
}
using TreeFn = void (*)(TreeParams);
template <typename TT, typename TQ>
void pick_tree2(bool logits, int N, TreeFn* f) {
  if (logits) {
    f[0] = tree_decide_kernel<TT, TQ, true>;
    f[1] = N <= 4 ? tree_walk_kernel<TT, TQ, true, 4> : tree_walk_kernel<TT, TQ, true, 8>;
  } else {
    f[0] = tree_decide_kernel<TT, TQ, false>;
    f[1] = N <= 4 ? tree_walk_kernel<TT, TQ, false, 4> : tree_walk_kernel<TT, TQ, false, 8>;
  }
}
void pick_tree(cosine_dtype_t tt, cosine_dtype_t tq, bool logits, int N, TreeFn* f) {
  if (tt == COSINE_BF16 && tq == COSINE_BF16) return pick_tree2<__nv_bfloat16, __nv_bfloat16>(logits, N, f);
  if (tt == COSINE_BF16 && tq == COSINE_F32) return pick_tree2<__nv_bfloat16, float>(logits, N, f);
  if (tt == COSINE_F32 && tq == COSINE_BF16) return pick_tree2<float, __nv_bfloat16>(logits, N, f);
  return pick_tree2<float, float>(logits, N, f);
}

void pick_split(cosine_dtype_t tt, cosine_dtype_t tq, bool logits, int N, SplitFn* f) {
  if (tt == COSINE_BF16 && tq == COSINE_BF16) return pick_split2<__nv_bfloat16, __nv_bfloat16>(logits, N, f);
  if (tt == COSINE_BF16 && tq == COSINE_F32) return pick_split2<__nv_bfloat16, float>(logits, N, f);
  if (tt == COSINE_F32 && tq == COSINE_BF16) return pick_split2<float, __nv_bfloat16>(logits, N, f);
  return pick_split2<float, float>(logits, N, f);
}
template <typename TT, typename TQ>
void pick_shard2(bool logits, int N, SplitFn* f) {
  if (logits) {
    f[0] = shard_pack_kernel<TT, TQ, true>;
    f[1] = shard_decide_kernel<true>;
    f[2] = N <= 4 ? shard_sample_kernel<TT, TQ, true, 4> : shard_sample_kernel<TT, TQ, true, 8>;
  } else {
    f[0] = shard_pack_kernel<TT, TQ, false>;
    f[1] = shard_decide_kernel<false>;
    f[2] = N <= 4 ? shard_sample_kernel<TT, TQ, false, 4> : shard_sample_kernel<TT, TQ, false, 8>;
  }
}
void pick_shard(cosine_dtype_t tt, cosine_dtype_t tq, bool logits, int N, SplitFn* f) {
  if (tt == COSINE_BF16 && tq == COSINE_BF16) return pick_shard2<__nv_bfloat16, __nv_bfloat16>(logits, N, f);
  if (tt == COSINE_BF16 && tq == COSINE_F32) return pick_shard2<__nv_bfloat16, float>(logits, N, f);
  if (tt == COSINE_F32 && tq == COSINE_BF16) return pick_shard2<float, __nv_bfloat16>(logits, N, f);
  return pick_shard2<float, float>(logits, N, f);
}
template <typename TT, typename TQ>
KernelFn pick_kernel2(bool logits, int N) {
  if (logits) return N <= 4 ? unit_kernel<TT, TQ, true, 4> : unit_kernel<TT, TQ, true, 8>;
  return N <= 4 ? unit_kernel<TT, TQ, false, 4> : unit_kernel<TT, TQ, false, 8>;
}
KernelFn pick_kernel(cosine_dtype_t tt, cosine_dtype_t tq, bool logits, int N) {
  if (tt == COSINE_BF16 && tq == COSINE_BF16) return pick_kernel2<__nv_bfloat16, __nv_bfloat16>(logits, N);
  if (tt == COSINE_BF16 && tq == COSINE_F32) return pick_kernel2<__nv_bfloat16, float>(logits, N);
  if (tt == COSINE_F32 && tq == COSINE_BF16) return pick_kernel2<float, __nv_bfloat16>(logits, N);
  return pick_kernel2<float, float>(logits, N);
}

}  // namespace cosine

// =====================================================================================
// C ABI
// =====================================================================================
using namespace cosine;

struct cosine_ctx_s {
  cosine_config_t cfg;
  int64_t V;
  UnitRec* recs = nullptr;
  PartRec* parts = nullptr;
  PosDec* pdec = nullptr;
  int32_t* counters = nullptr;
  NodeDec* ndec = nullptr;
  ChildPQ* cpq = nullptr;
  double* segsum = nullptr;
  size_t segsum_cap = 0;
  cudaStream_t aux = nullptr;
  cudaEvent_t ev[kMaxChunks + 1] = {};
  // optional live timing of the dominant kernel (stats_kernel) with CUDA events on the stream
  int prof_on = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev;
  size_t prof_n = 0;
  int32_t* done = nullptr;
  int32_t* first_rej = nullptr;
  std::string err;
  int32_t last_launches = 0;
  int32_t last_cluster = 0, last_ncl = 0;
  int32_t* lz = nullptr;  // lazy verification: per-request state
  size_t parts_cap = 0;    // PartRec entries in `parts`
  // vocabulary-sharded mode (nranks > 1)
  ncclComm_t comm = nullptr;
  uint32_t* rec_send = nullptr;
  uint32_t* rec_all = nullptr;
  double* zsend = nullptr;
  double* zall = nullptr;
  YRec* ysend = nullptr;
  YRec* yall = nullptr;
};

static thread_local std::string g_init_error;

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

cosine_status_t fail(cosine_ctx_t ctx, cosine_status_t s, const std::string& msg) {
  if (ctx) ctx->err = msg;
  else g_init_error = msg;
  return s;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
size_t esize(cosine_dtype_t t) { return t == COSINE_BF16 ? 2 : 4; }

int pick_cluster(const cosine_ctx_t ctx, int64_t units, int64_t ngroups) {
  if (ctx->cfg.cluster_size > 0) return std::min(ctx->cfg.cluster_size, 8);
  // ~8 groups (64 elements per row) per thread, then widen while the grid is small
  int C = 1;
  while (C < 8 && ngroups > (int64_t)C * kThreads * 8) C *= 2;
  while (C < 8 && units * C < 148 * 8 && ngroups >= (int64_t)C * 2 * kThreads) C *= 2;
  return C;
}

cosine_status_t launch(cosine_ctx_t ctx, cudaStream_t stream, Params& P, int64_t units,
                       cosine_dtype_t tt, cosine_dtype_t tq, bool logits) {
  const int C = pick_cluster(ctx, units, P.ngroups);
  P.C = C;
  P.gpc = (P.ngroups + C - 1) / C;
  P.recs = ctx->recs;
  P.done = ctx->done;
  P.first_rej = ctx->first_rej;
  if (units == 0) { ctx->last_launches = 0; return COSINE_OK; }
  KernelFn fn = pick_kernel(tt, tq, logits, P.N);
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.gridDim = dim3((unsigned)(units * C), 1, 1);
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.dynamicSmemBytes = 0;
  lc.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, fn, P);
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = 1;
  return COSINE_OK;
}

// Kernel A (stats + decisions) then kernel B (first rejection + cooperative sample), the
// latter launched with programmatic dependent launch so its launch overlaps A's tail.
// Tiles (256 groups) per resample CTA: fewer -> more, shorter CTAs (less wave tail).
int resample_tiles_per_cta() {
  int t = 8;
  if (const char* v = getenv("COSINE_TPC")) t = atoi(v);
  return std::max(1, std::min(kSegTilesPerCta, t));
}

cosine_status_t launch_split(cosine_ctx_t ctx, cudaStream_t stream, SplitParams& S,
                             cosine_dtype_t tt, cosine_dtype_t tq, bool logits) {
  SplitFn fn[3];
  pick_split(tt, tq, logits, S.N, fn);
  const int64_t units = (int64_t)S.B * (S.k + 1);
  // kernel A: ~8 groups (64 elements per row) per thread, at least ~8 CTAs per SM of work
  int C = 1;
  if (ctx->cfg.cluster_size > 0) {
    C = ctx->cfg.cluster_size;
  } else {
    while (C < kMaxC && S.ngroups > (int64_t)C * kThreads * 8) C *= 2;
    while (C < kMaxC && units * C < 148 * 8 && S.ngroups >= (int64_t)C * 2 * kThreads) C *= 2;
  }
  S.C = C;
  S.cg = (S.ngroups + C - 1) / C;
  S.nseg = (S.ngroups + kTileGroups - 1) / kTileGroups;
  S.tpc = resample_tiles_per_cta();
  S.spr = (int)((S.nseg + S.tpc - 1) / S.tpc);
  S.parts = ctx->parts;
  S.pdec = ctx->pdec;
  S.segsum = ctx->segsum;
  S.counters = ctx->counters;
  if ((size_t)S.B * (size_t)S.nseg > ctx->segsum_cap)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "segment scratch too small");
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  // Batch pipelining (experiment, COSINE_CHUNKS=n): the requests are split into n slices; slice
  // c's statistics stream on `stream` while the decisions + final draws of slice c-1 run on the
  // high-priority aux stream (fork / join by events, capturable in a CUDA graph).  Measured on
  // c3 (profiles/r1_ncu_summary.md): 1 slice 486 us, 2 -> 502, 4 -> 527, 8 -> 630 — every slice
  // boundary adds a stats-kernel tail, more than the hidden B phase saves — so the default is 1.
  int nch = 1;
  if (const char* ev = getenv("COSINE_CHUNKS")) nch = atoi(ev);
  nch = std::max(1, std::min(nch, std::min(kMaxChunks - 1, S.B)));
  const int cb = (S.B + nch - 1) / nch;
  nch = (S.B + cb - 1) / cb;
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  if (ctx->prof_on) {
    if (ctx->prof_n == ctx->prof_ev.size()) {
      cudaEvent_t a0, a1;
      cudaEventCreate(&a0);
      cudaEventCreate(&a1);
      ctx->prof_ev.emplace_back(a0, a1);
    }
    pe0 = ctx->prof_ev[ctx->prof_n].first;
    pe1 = ctx->prof_ev[ctx->prof_n].second;
    ctx->prof_n++;
    cudaEventRecord(pe0, stream);
  }
  cudaError_t e = cudaSuccess;
  int launches = 0;
  const char* nofuse = getenv("COSINE_NOFUSE");
  if (nch == 1 && nofuse && nofuse[0] == '1') {  // (experiment) kernel A -> B1 -> B2 with PDL
    S.b_off = 0;
    S.nb = S.B;
    lc.gridDim = dim3((unsigned)(units * C), 1, 1);
    e = cudaLaunchKernelEx(&lc, fn[0], S);
    if (pe1) cudaEventRecord(pe1, stream);
    if (e == cudaSuccess) {
      lc.gridDim = dim3((unsigned)((units + kWarps - 1) / kWarps), 1, 1);
      lc.attrs = pe1 ? nullptr : at;
      lc.numAttrs = pe1 ? 0 : 1;
      e = cudaLaunchKernelEx(&lc, fn[1], S);
    }
    if (e == cudaSuccess) {
      lc.gridDim = dim3((unsigned)(S.B * S.spr), 1, 1);
      lc.attrs = at;
      lc.numAttrs = 1;
      e = cudaLaunchKernelEx(&lc, fn[2], S);
    }
    launches = 3;
  } else if (nch == 1) {
    // A -> B1 -> B2, each a programmatic dependent of the previous one: B1 / B2 CTAs are
    // scheduled into the previous grid's tail wave and wait per unit / per request (counters)
    S.b_off = 0;
    S.nb = S.B;
    S.fused = 1;
    S.dcnt = ctx->counters + std::max(ctx->cfg.max_batch, 1);
    S.ucnt = ctx->counters + 2 * (size_t)std::max(ctx->cfg.max_batch, 1);
    lc.gridDim = dim3((unsigned)(units * C), 1, 1);
    e = cudaLaunchKernelEx(&lc, fn[0], S);  // kernel A
    if (pe1) cudaEventRecord(pe1, stream);
    if (e == cudaSuccess) {  // kernel B1 (decisions)
      lc.gridDim = dim3((unsigned)((units + kWarps - 1) / kWarps), 1, 1);
      lc.attrs = pe1 ? nullptr : at;  // (an event record between the two breaks PDL)
      lc.numAttrs = pe1 ? 0 : 1;
      e = cudaLaunchKernelEx(&lc, fn[1], S);
    }
    if (e == cudaSuccess) {  // kernel B2 (first rejection + resample)
      lc.gridDim = dim3((unsigned)(S.B * S.spr), 1, 1);
      lc.attrs = at;
      lc.numAttrs = 1;
      e = cudaLaunchKernelEx(&lc, fn[2], S);
    }
    launches = 3;
  } else {
    e = cudaEventRecord(ctx->ev[0], stream);  // fork: aux waits for the work already on `stream`
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->aux, ctx->ev[0], 0);
    cudaLaunchConfig_t lb = lc;
    lb.stream = ctx->aux;
    for (int c = 0; c < nch && e == cudaSuccess; ++c) {
      S.b_off = c * cb;
      S.nb = std::min(cb, S.B - S.b_off);
      const int64_t cu = (int64_t)S.nb * (S.k + 1);
      lc.gridDim = dim3((unsigned)(cu * C), 1, 1);
      lc.attrs = nullptr;
      lc.numAttrs = 0;
      e = cudaLaunchKernelEx(&lc, fn[0], S);  // kernel A of slice c on `stream`
      if (e == cudaSuccess) e = cudaEventRecord(ctx->ev[c + 1], stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->aux, ctx->ev[c + 1], 0);
      if (e == cudaSuccess) {  // B1 + B2 of slice c on aux
        lb.gridDim = dim3((unsigned)((cu + kWarps - 1) / kWarps), 1, 1);
        lb.attrs = nullptr;
        lb.numAttrs = 0;
        e = cudaLaunchKernelEx(&lb, fn[1], S);
      }
      if (e == cudaSuccess) {
        lb.gridDim = dim3((unsigned)(S.nb * S.spr), 1, 1);
        lb.attrs = at;
        lb.numAttrs = 1;
        e = cudaLaunchKernelEx(&lb, fn[2], S);
      }
      launches += 3;
    }
    if (pe1 && e == cudaSuccess) cudaEventRecord(pe1, stream);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev[kMaxChunks], ctx->aux);  // join
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, ctx->ev[kMaxChunks], 0);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("verify kernels: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = launches;
  ctx->last_cluster = C;
  return COSINE_OK;
}

// Vocabulary-sharded verification (cosine_shard.cuh): 7 kernels and 3 all-gathers on `stream`.
cosine_status_t launch_shard(cosine_ctx_t ctx, cudaStream_t stream, SplitParams& S, cosine_dtype_t tt,
                             cosine_dtype_t tq, bool logits) {
  SplitFn fa[3], fs[3];
  pick_split(tt, tq, logits, S.N, fa);
  pick_shard(tt, tq, logits, S.N, fs);
  const int64_t units = (int64_t)S.B * (S.k + 1);
  int C = 1;
  if (ctx->cfg.cluster_size > 0) {
    C = ctx->cfg.cluster_size;
  } else {
    while (C < kMaxC && S.ngroups > (int64_t)C * kThreads * 8) C *= 2;
    while (C < kMaxC && units * C < 148 * 8 && S.ngroups >= (int64_t)C * 2 * kThreads) C *= 2;
  }
  S.C = C;
  S.cg = (S.ngroups + C - 1) / C;
  S.nseg = (S.ngroups + kTileGroups - 1) / kTileGroups;
  S.tpc = resample_tiles_per_cta();
  S.spr = (int)((S.nseg + S.tpc - 1) / S.tpc);
  S.parts = ctx->parts;
  S.pdec = ctx->pdec;
  S.segsum = ctx->segsum;
  S.counters = ctx->counters;
  S.b_off = 0;
  S.nb = S.B;
  S.shard = 1;
  S.G = ctx->cfg.nranks;
  S.rank = ctx->cfg.rank;
  S.v0 = ctx->cfg.vocab_begin;
  S.Vg = ctx->cfg.vocab_size;
  S.rec_words = shard_rec_words(S.N);
  S.rec_send = ctx->rec_send;
  S.rec_all = ctx->rec_all;
  S.zsend = ctx->zsend;
  S.zall = ctx->zall;
  S.ysend = ctx->ysend;
  S.yall = ctx->yall;
  if ((size_t)S.B * (size_t)S.nseg > ctx->segsum_cap)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "segment scratch too small");
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  const unsigned unit_blocks = (unsigned)((units + kWarps - 1) / kWarps);
  auto launch = [&](SplitFn f, unsigned grid, bool pdl) {
    lc.gridDim = dim3(grid, 1, 1);
    lc.attrs = pdl ? at : nullptr;
    lc.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&lc, f, S);
  };
  const char* stage = "stats";
  cudaEvent_t pe1 = nullptr;
  if (ctx->prof_on) {  // live timing of the dominant kernel (as in launch_split)
    if (ctx->prof_n == ctx->prof_ev.size()) {
      cudaEvent_t a0, a1;
      cudaEventCreate(&a0);
      cudaEventCreate(&a1);
      ctx->prof_ev.emplace_back(a0, a1);
    }
    cudaEventRecord(ctx->prof_ev[ctx->prof_n].first, stream);
    pe1 = ctx->prof_ev[ctx->prof_n].second;
    ctx->prof_n++;
  }
  cudaError_t e = launch(fa[0], (unsigned)(units * C), false);  // local row statistics
  if (pe1) cudaEventRecord(pe1, stream);
  if (e == cudaSuccess) { stage = "pack"; e = launch(fs[0], unit_blocks, pe1 == nullptr); }
  ncclResult_t r = ncclSuccess;
  if (e == cudaSuccess) {
    r = ncclAllGather(ctx->rec_send, ctx->rec_all, (size_t)units * S.rec_words * 4, ncclUint8, ctx->comm, stream);
  }
  if (e == cudaSuccess && r == ncclSuccess) { stage = "decide"; e = launch(fs[1], unit_blocks, false); }
  if (e == cudaSuccess && r == ncclSuccess) { stage = "resample"; e = launch(fa[2], (unsigned)(S.B * S.spr), false); }
  if (e == cudaSuccess && r == ncclSuccess)
    r = ncclAllGather(ctx->zsend, ctx->zall, (size_t)S.B * sizeof(double), ncclUint8, ctx->comm, stream);
  if (e == cudaSuccess && r == ncclSuccess) { stage = "sample"; e = launch(fs[2], (unsigned)S.B, false); }
  if (e == cudaSuccess && r == ncclSuccess)
    r = ncclAllGather(ctx->ysend, ctx->yall, (size_t)S.B * sizeof(YRec), ncclUint8, ctx->comm, stream);
  if (e == cudaSuccess && r == ncclSuccess) {
    stage = "finish";
    lc.gridDim = dim3((unsigned)((S.B + kThreads - 1) / kThreads), 1, 1);
    lc.attrs = nullptr;
    lc.numAttrs = 0;
    e = cudaLaunchKernelEx(&lc, shard_finish_kernel, S);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("sharded verify (") + stage + "): " + cudaGetErrorString(e));
  }
  if (r != ncclSuccess) {
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_NCCL, std::string("sharded verify all-gather: ") + ncclGetErrorString(r));
  }
  ctx->last_launches = 7;
  ctx->last_cluster = C;
  return COSINE_OK;
}

using LazyFn = void (*)(SplitParams);
template <typename TT, typename TQ>
LazyFn pick_lazy2(bool logits) {
  return logits ? lazy_decide_kernel<TT, TQ, true> : lazy_decide_kernel<TT, TQ, false>;
}
LazyFn pick_lazy(cosine_dtype_t tt, cosine_dtype_t tq, bool logits) {
  if (tt == COSINE_BF16 && tq == COSINE_BF16) return pick_lazy2<__nv_bfloat16, __nv_bfloat16>(logits);
  if (tt == COSINE_BF16 && tq == COSINE_F32) return pick_lazy2<__nv_bfloat16, float>(logits);
  if (tt == COSINE_F32 && tq == COSINE_BF16) return pick_lazy2<float, __nv_bfloat16>(logits);
  return pick_lazy2<float, float>(logits);
}

// Lazy verification (NEXT-1): rounds r = 0..k of (stats of position r of the requests still
// verifying -> their decisions), then the final draws.  2 (k + 1) + 1 launches on `stream`.
cosine_status_t launch_lazy(cosine_ctx_t ctx, cudaStream_t stream, SplitParams& S, cosine_dtype_t tt,
                            cosine_dtype_t tq, bool logits) {
  SplitFn fn[3];
  pick_split(tt, tq, logits, S.N, fn);
  const LazyFn fd = pick_lazy(tt, tq, logits);
  int C = 1;
  if (ctx->cfg.cluster_size > 0) {
    C = ctx->cfg.cluster_size;
  } else {
    while (C < kMaxC && S.ngroups > (int64_t)C * kThreads * 8) C *= 2;
    while (C < kMaxC && (int64_t)S.B * C < 148 * 8 && S.ngroups >= (int64_t)C * 2 * kThreads) C *= 2;
  }
  S.C = C;
  S.cg = (S.ngroups + C - 1) / C;
  S.nseg = (S.ngroups + kTileGroups - 1) / kTileGroups;
  S.tpc = resample_tiles_per_cta();
  S.spr = (int)((S.nseg + S.tpc - 1) / S.tpc);
  S.parts = ctx->parts;
  S.pdec = ctx->pdec;
  S.segsum = ctx->segsum;
  S.counters = ctx->counters;
  S.b_off = 0;
  S.nb = S.B;
  S.lz = ctx->lz;
  if ((size_t)S.B * (size_t)S.nseg > ctx->segsum_cap)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "segment scratch too small");
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaError_t e = cudaSuccess;
  int launches = 0;
  // round shape (measured, c3): C chunk CTAs per unit in the first round; later rounds stream
  // fewer requests, so more CTAs per unit (COSINE_LAZY_C); `span` positions per round
  // (COSINE_LAZY_SPAN) trade speculative bytes for fewer dependent rounds
  int C1 = C, span = 2;  // c3: span 1 -> 393 us, 2 -> 366 us, 3 -> 372 us
  if (const char* v = getenv("COSINE_LAZY_C")) C1 = std::max(1, std::min(kMaxC, atoi(v)));
  if (const char* v = getenv("COSINE_LAZY_SPAN")) span = std::max(1, std::min(S.k + 1, atoi(v)));
  S.lazy_span = span;
  // per-unit counters: each round's decide kernel is scheduled into the stats tail (PDL) and
  // waits per position (COSINE_LAZY_FUSED=0: whole-grid waits)
  S.fused = 1;
  if (const char* v = getenv("COSINE_LAZY_FUSED")) S.fused = atoi(v) != 0;
  S.dcnt = ctx->counters + std::max(ctx->cfg.max_batch, 1);
  S.ucnt = ctx->counters + 2 * (size_t)std::max(ctx->cfg.max_batch, 1);
  int span0 = span;  // the first round's span (COSINE_LAZY_SPAN0)
  if (const char* v = getenv("COSINE_LAZY_SPAN0")) span0 = std::max(1, std::min(S.k + 1, atoi(v)));
  for (int r = 0; r <= S.k && e == cudaSuccess; r += S.lazy_span) {
    S.lazy_span = (r == 0) ? span0 : span;
    S.lazy = r + 1;
    S.C = (r == 0) ? C : C1;
    S.cg = (S.ngroups + S.C - 1) / S.C;
    lc.gridDim = dim3((unsigned)((int64_t)S.B * S.lazy_span * S.C), 1, 1);
    lc.attrs = nullptr;  // stream order: the round reads the previous round's lz
    lc.numAttrs = 0;
    e = cudaLaunchKernelEx(&lc, fn[0], S);
    if (e == cudaSuccess) {
      lc.gridDim = dim3((unsigned)((S.B + kWarps - 1) / kWarps), 1, 1);
      lc.attrs = at;
      lc.numAttrs = 1;
      e = cudaLaunchKernelEx(&lc, fd, S);
    }
    launches += 2;
  }
  S.lazy = 0;
  S.fused = 0;  // the final draws wait for the last round's grid (griddepcontrol.wait)
  if (e == cudaSuccess) {
    lc.gridDim = dim3((unsigned)(S.B * S.spr), 1, 1);
    lc.attrs = at;
    lc.numAttrs = 1;
    e = cudaLaunchKernelEx(&lc, fn[2], S);
    launches += 1;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("lazy verify kernels: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = launches;
  ctx->last_cluster = C;
  return COSINE_OK;
}

void fill_common(Params& P, const cosine_ctx_t ctx, int B, int k, int N, float T) {
  memset(&P, 0, sizeof(P));
  P.B = B;
  P.k = k;
  P.N = N;
  P.V = ctx->V;
  P.ngroups = (ctx->V + kGroup - 1) / kGroup;
  P.gfull = ctx->V / kGroup;
  P.T = T;
  P.greedy = (T == 0.f);
  const double k2 = (T > 0.f) ? 1.4426950408889634 / (double)T : 0.0;
  P.k2d = k2;
  P.k2f = (float)k2;
  P.seed = ctx->cfg.seed;
}

cosine_status_t check_rows(cosine_ctx_t ctx, const void* p, int64_t ld, cosine_dtype_t t,
                           const char* what) {
  if (!p) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, std::string(what) + " is NULL");
  if (ld < ctx->V) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, std::string(what) + ": ld < vocabulary width");
  if (!aligned16(p) || ((uint64_t)ld * esize(t)) % 16 != 0)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, std::string(what) + ": rows must be 16-byte aligned");
  return COSINE_OK;
}

cosine_status_t check_common(cosine_ctx_t ctx, int B, int k, int N) {
  if (!ctx) return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "NULL context");
  if (B < 0 || B > ctx->cfg.max_batch) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "B outside [0, max_batch]");
  if (k < 1 || k > ctx->cfg.max_draft_len) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "k outside [1, max_draft_len]");
  if (N < 1 || N > ctx->cfg.max_drafters || N > kMaxN) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "N outside [1, max_drafters]");
  return COSINE_OK;
}

}  // namespace

extern "C" {

cosine_status_t cosine_verify_init(const cosine_config_t* cfg, cosine_ctx_t* out) {
  if (!out) return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!cfg) return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "cfg is NULL");
  if (cfg->vocab_size < 1 || cfg->vocab_begin < 0 || cfg->vocab_end > cfg->vocab_size ||
      cfg->vocab_end <= cfg->vocab_begin)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "bad vocabulary range");
  if (cfg->vocab_end - cfg->vocab_begin > (int64_t)0x7fffffff)
    return fail(nullptr, COSINE_ERR_UNSUPPORTED, "vocabulary wider than 2^31 - 1");
  if (cfg->max_tree_nodes < 0 || cfg->max_tree_nodes > kTreeMaxNodes)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "max_tree_nodes outside [0, 1024]");
  if (cfg->max_batch < 0 || cfg->max_draft_len < 1 || cfg->max_draft_len > kMaxPos - 1 ||
      cfg->max_drafters < 1 || cfg->max_drafters > kMaxN)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "bad max_* sizes (max_draft_len <= 64, max_drafters <= 8)");
  if ((cfg->target_dtype != COSINE_BF16 && cfg->target_dtype != COSINE_F32) ||
      (cfg->draft_dtype != COSINE_BF16 && cfg->draft_dtype != COSINE_F32))
    return fail(nullptr, COSINE_ERR_UNSUPPORTED, "dtype must be COSINE_BF16 or COSINE_F32");
  if (cfg->draft_kind != COSINE_DRAFT_PROBS && cfg->draft_kind != COSINE_DRAFT_LOGITS)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "bad draft_kind");
  if (cfg->nranks < 1 || cfg->nranks > 32 || cfg->rank < 0 || cfg->rank >= cfg->nranks)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "nranks must be in [1, 32] and rank in [0, nranks)");
  if (cfg->nranks == 1 && (cfg->vocab_begin != 0 || cfg->vocab_end != cfg->vocab_size))
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "an unsharded context covers [0, vocab_size)");
  if (cfg->nranks > 1 && !cfg->nccl_unique_id)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "nranks > 1 needs nccl_unique_id (cosine_nccl_unique_id on rank 0)");
  if (cfg->cluster_size != 0 && cfg->cluster_size != 1 && cfg->cluster_size != 2 &&
      cfg->cluster_size != 4 && cfg->cluster_size != 8 && cfg->cluster_size != 16)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "cluster_size must be 0, 1, 2, 4, 8 or 16");
  cosine_ctx_t ctx = new (std::nothrow) cosine_ctx_s();
  if (!ctx) return fail(nullptr, COSINE_ERR_OUT_OF_MEMORY, "host allocation failed");
  ctx->cfg = *cfg;
  ctx->cfg.nccl_unique_id = nullptr;
  ctx->V = cfg->vocab_end - cfg->vocab_begin;
  DeviceGuard dg(cfg->device);
  const size_t nb = (size_t)std::max(cfg->max_batch, 1);
  cudaError_t e = cudaMalloc(&ctx->recs, nb * (size_t)(cfg->max_draft_len + 1) * sizeof(UnitRec));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->done, nb * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->first_rej, nb * sizeof(int32_t));
  const size_t nu = nb * (size_t)std::max(cfg->max_draft_len + 1, std::max(cfg->max_tree_nodes, 1));
  const size_t nt = nb * (size_t)std::max(cfg->max_tree_nodes, 1);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->ndec, nt * sizeof(NodeDec));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->cpq, nt * sizeof(ChildPQ));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->parts, nu * kMaxC * sizeof(PartRec));
  ctx->parts_cap = nu * kMaxC;
  if (e == cudaSuccess) e = cudaMalloc(&ctx->pdec, nu * sizeof(PosDec));
  // counters: [B] kernel-B CTAs per request | [B] decided units per request | [B][k+1] chunks per unit
  const size_t ncnt = 2 * nb + nb * (size_t)(cfg->max_draft_len + 1);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->counters, ncnt * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->lz, nb * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemset(ctx->counters, 0, ncnt * sizeof(int32_t));
  ctx->segsum_cap = nb * (size_t)((ctx->V + (int64_t)kTileElems - 1) / kTileElems);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->segsum, ctx->segsum_cap * sizeof(double));
  if (e == cudaSuccess) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    e = cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, hi);
  }
  for (int j = 0; j <= kMaxChunks && e == cudaSuccess; ++j)
    e = cudaEventCreateWithFlags(&ctx->ev[j], cudaEventDisableTiming);
  if (e == cudaSuccess) {
    init_scratch<<<(unsigned)((nb + 255) / 256), 256>>>(ctx->done, ctx->first_rej, (int)nb);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && cfg->nranks > 1) {  // vocabulary-sharded: exchange buffers + communicator
    const size_t units = nb * (size_t)(cfg->max_draft_len + 1);
    const size_t rb = units * (size_t)shard_rec_words(cfg->max_drafters) * 4;
    e = cudaMalloc(&ctx->rec_send, rb);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->rec_all, rb * (size_t)cfg->nranks);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->zsend, nb * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&ctx->zall, nb * sizeof(double) * (size_t)cfg->nranks);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->ysend, nb * sizeof(YRec));
    if (e == cudaSuccess) e = cudaMalloc(&ctx->yall, nb * sizeof(YRec) * (size_t)cfg->nranks);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  ncclResult_t nr = ncclSuccess;
  if (e == cudaSuccess && cfg->nranks > 1) {
    ncclUniqueId uid;
    memcpy(&uid, cfg->nccl_unique_id, sizeof(uid));
    nr = ncclCommInitRank(&ctx->comm, cfg->nranks, uid, cfg->rank);
    if (nr != ncclSuccess) ctx->comm = nullptr;
  }
  if (e != cudaSuccess || nr != ncclSuccess) {
    std::string msg = (e != cudaSuccess) ? std::string("init: ") + cudaGetErrorString(e)
                                         : std::string("init: ncclCommInitRank: ") + ncclGetErrorString(nr);
    cudaFree(ctx->rec_send);
    cudaFree(ctx->rec_all);
    cudaFree(ctx->zsend);
    cudaFree(ctx->zall);
    cudaFree(ctx->ysend);
    cudaFree(ctx->yall);
    cudaFree(ctx->lz);
    cudaGetLastError();
    cudaFree(ctx->recs);
    cudaFree(ctx->done);
    cudaFree(ctx->first_rej);
    cudaFree(ctx->parts);
    cudaFree(ctx->pdec);
    cudaFree(ctx->counters);
    cudaFree(ctx->ndec);
    cudaFree(ctx->cpq);
    cudaFree(ctx->segsum);
    for (int j = 0; j <= kMaxChunks; ++j)
      if (ctx->ev[j]) cudaEventDestroy(ctx->ev[j]);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    delete ctx;
    if (e == cudaSuccess) return fail(nullptr, COSINE_ERR_NCCL, msg);
    return fail(nullptr, e == cudaErrorMemoryAllocation ? COSINE_ERR_OUT_OF_MEMORY : COSINE_ERR_CUDA, msg);
  }
  *out = ctx;
  return COSINE_OK;
}

cosine_status_t cosine_verify_destroy(cosine_ctx_t ctx) {
  if (!ctx) return COSINE_OK;
  DeviceGuard dg(ctx->cfg.device);
  cudaDeviceSynchronize();
  cudaFree(ctx->recs);
  cudaFree(ctx->done);
  cudaFree(ctx->first_rej);
  cudaFree(ctx->parts);
  cudaFree(ctx->pdec);
  cudaFree(ctx->counters);
  cudaFree(ctx->ndec);
  cudaFree(ctx->cpq);
  cudaFree(ctx->segsum);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  cudaFree(ctx->lz);
  cudaFree(ctx->rec_send);
  cudaFree(ctx->rec_all);
  cudaFree(ctx->zsend);
  cudaFree(ctx->zall);
  cudaFree(ctx->ysend);
  cudaFree(ctx->yall);
  for (int j = 0; j <= kMaxChunks; ++j)
    if (ctx->ev[j]) cudaEventDestroy(ctx->ev[j]);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  for (auto& pe : ctx->prof_ev) {
    cudaEventDestroy(pe.first);
    cudaEventDestroy(pe.second);
  }
  delete ctx;
  return COSINE_OK;
}

cosine_status_t cosine_nccl_unique_id(void* out, int64_t capacity) {
  if (!out || capacity < (int64_t)sizeof(ncclUniqueId))
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "unique id buffer smaller than COSINE_NCCL_UNIQUE_ID_BYTES");
  ncclUniqueId uid;
  const ncclResult_t r = ncclGetUniqueId(&uid);
  if (r != ncclSuccess) return fail(nullptr, COSINE_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  memcpy(out, &uid, sizeof(uid));
  return COSINE_OK;
}

const char* cosine_last_error(cosine_ctx_t ctx) {
  return ctx ? ctx->err.c_str() : g_init_error.c_str();
}

int32_t cosine_last_launch_count(cosine_ctx_t ctx) { return ctx ? ctx->last_launches : 0; }

cosine_status_t cosine_profile_enable(cosine_ctx_t ctx, int32_t enable) {
  if (!ctx) return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "NULL context");
  ctx->prof_on = enable ? 1 : 0;
  ctx->prof_n = 0;
  return COSINE_OK;
}

cosine_status_t cosine_profile_read(cosine_ctx_t ctx, double* total_ms, int32_t* launches) {
  if (!ctx || !total_ms || !launches) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard dg(ctx->cfg.device);
  double t = 0.0;
  for (size_t j = 0; j < ctx->prof_n; ++j) {
    float ms = 0.f;
    if (cudaEventSynchronize(ctx->prof_ev[j].second) != cudaSuccess ||
        cudaEventElapsedTime(&ms, ctx->prof_ev[j].first, ctx->prof_ev[j].second) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, COSINE_ERR_CUDA, "profile events not recorded");
    }
    t += ms;
  }
  *total_ms = t;
  *launches = (int32_t)ctx->prof_n;
  ctx->prof_n = 0;
  return COSINE_OK;
}

cosine_status_t cosine_fuse_drafts(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t k,
                                   int32_t N, const void* draft, int64_t ld_q,
                                   const int32_t* draft_tokens, const uint64_t* request_ids,
                                   uint32_t step, float temperature,
                                   cosine_weight_mode_t weight_mode, cosine_select_mode_t select_mode,
                                   int32_t* fused_tokens, float* weights, float* draft_norm,
                                   float* fused_q, int64_t ld_fq, int32_t* status) {
  cosine_status_t s = check_common(ctx, B, k, N);
  if (s != COSINE_OK) return s;
  if (ctx->cfg.nranks > 1)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "cosine_fuse_drafts runs on unsharded contexts (nranks == 1)");
  if (B == 0) { ctx->last_launches = 0; return COSINE_OK; }
  if ((s = check_rows(ctx, draft, ld_q, ctx->cfg.draft_dtype, "draft")) != COSINE_OK) return s;
  if (!draft_tokens || !request_ids || !fused_tokens || !status)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "NULL required pointer");
  if ((int)weight_mode < 0 || (int)weight_mode > 3 || (int)select_mode < 0 || (int)select_mode > 1)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "bad weight / select mode");
  if (weight_mode == COSINE_W_POINT && select_mode == COSINE_SEL_SAMPLE)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "POINT weights need ARGMAX selection");
  if (ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS && !(temperature > 0.f && std::isfinite(temperature)))
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "LOGITS drafts need temperature > 0");
  if (fused_q && (ld_fq < ctx->V || !aligned16(fused_q) || (ld_fq * 4) % 16 != 0))
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "fused_q must be 16-byte aligned with ld_fq >= V");
  DeviceGuard dg(ctx->cfg.device);
  Params P;
  fill_common(P, ctx, B, k, N, ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS ? temperature : 1.f);
  P.greedy = 0;
  P.mode = kModeFuse;
  P.ld_q = ld_q;
  P.ld_fq = ld_fq;
  P.draft = draft;
  P.draft_tokens = draft_tokens;
  P.rids = request_ids;
  P.step = step;
  P.weight_mode = weight_mode;
  P.select_mode = select_mode;
  P.fused_tokens = fused_tokens;
  P.w_out = weights;
  P.norm_out = draft_norm;
  P.fused_q = fused_q;
  P.status = status;
  return launch(ctx, (cudaStream_t)stream, P, (int64_t)B * k, ctx->cfg.target_dtype,
                ctx->cfg.draft_dtype, ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS);
}

cosine_status_t cosine_verify_batch(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t k,
                                    int32_t N, const void* target_logits, int64_t ld_t,
                                    float temperature, const void* draft, int64_t ld_q,
                                    const int32_t* draft_tokens, const int32_t* draft_len,
                                    const uint64_t* request_ids, uint32_t step,
                                    cosine_weight_mode_t weight_mode,
                                    cosine_select_mode_t select_mode, int32_t* accept_len,
                                    int32_t* out_tokens, int32_t* status,
                                    const cosine_debug_t* debug) {
  cosine_status_t s = check_common(ctx, B, k, N);
  if (s != COSINE_OK) return s;
  if (B == 0) { ctx->last_launches = 0; return COSINE_OK; }
  if ((s = check_rows(ctx, target_logits, ld_t, ctx->cfg.target_dtype, "target_logits")) != COSINE_OK) return s;
  if ((s = check_rows(ctx, draft, ld_q, ctx->cfg.draft_dtype, "draft")) != COSINE_OK) return s;
  if (!draft_tokens || !request_ids || !accept_len || !out_tokens || !status)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "NULL required pointer");
  if (!(temperature >= 0.f) || !std::isfinite(temperature))
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "temperature must be finite and >= 0");
  if ((int)weight_mode < 0 || (int)weight_mode > 3 || (int)select_mode < 0 || (int)select_mode > 1)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "bad weight / select mode");
  if (weight_mode == COSINE_W_POINT && select_mode == COSINE_SEL_SAMPLE)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "POINT weights need ARGMAX selection");
  if (temperature == 0.f && (ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS || select_mode == COSINE_SEL_SAMPLE))
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "greedy (T = 0) needs PROBS drafts and ARGMAX selection");
  DeviceGuard dg(ctx->cfg.device);
  Params P;
  fill_common(P, ctx, B, k, N, temperature);
  P.mode = kModeVerify;
  P.ld_t = ld_t;
  P.ld_q = ld_q;
  P.target = target_logits;
  P.draft = draft;
  P.draft_tokens = draft_tokens;
  P.draft_len = draft_len;
  P.rids = request_ids;
  P.step = step;
  P.weight_mode = weight_mode;
  P.select_mode = select_mode;
  P.accept_len = accept_len;
  P.out_tokens = out_tokens;
  P.status = status;
  if (debug) P.dbg = *debug;
  const char* force_v2 = getenv("COSINE_FORCE_CLUSTER_KERNEL");
  if (ctx->cfg.nranks > 1) {  // vocabulary-sharded (cosine_shard.cuh)
    if (select_mode != COSINE_SEL_ARGMAX)
      return fail(ctx, COSINE_ERR_UNSUPPORTED, "vocabulary sharding takes ARGMAX selection");
    SplitParams S;
    memset(&S, 0, sizeof(S));
    S.B = B; S.k = k; S.N = N;
    S.V = P.V; S.ld_t = ld_t; S.ld_q = ld_q; S.ngroups = P.ngroups; S.gfull = P.gfull;
    S.k2f = P.k2f; S.k2d = P.k2d; S.greedy = P.greedy; S.weight_mode = weight_mode;
    S.target = target_logits; S.draft = draft; S.draft_tokens = draft_tokens; S.draft_len = draft_len;
    S.rids = request_ids; S.seed = P.seed; S.step = step;
    S.accept_len = accept_len; S.out_tokens = out_tokens; S.status = status; S.dbg = P.dbg;
    return launch_shard(ctx, (cudaStream_t)stream, S, ctx->cfg.target_dtype, ctx->cfg.draft_dtype,
                        ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS);
  }
  if (select_mode == COSINE_SEL_ARGMAX && !(force_v2 && force_v2[0] == '1')) {
    SplitParams S;
    memset(&S, 0, sizeof(S));
    S.B = B; S.k = k; S.N = N;
    S.V = P.V; S.ld_t = ld_t; S.ld_q = ld_q; S.ngroups = P.ngroups; S.gfull = P.gfull;
    S.k2f = P.k2f; S.k2d = P.k2d; S.greedy = P.greedy; S.weight_mode = weight_mode;
    S.target = target_logits; S.draft = draft; S.draft_tokens = draft_tokens; S.draft_len = draft_len;
    S.rids = request_ids; S.seed = P.seed; S.step = step;
    S.accept_len = accept_len; S.out_tokens = out_tokens; S.status = status; S.dbg = P.dbg;
    return launch_split(ctx, (cudaStream_t)stream, S, ctx->cfg.target_dtype, ctx->cfg.draft_dtype,
                        ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS);
  }
  return launch(ctx, (cudaStream_t)stream, P, (int64_t)B * (k + 1), ctx->cfg.target_dtype,
                ctx->cfg.draft_dtype, ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS);
}

cosine_status_t cosine_verify_batch_lazy(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t k,
                                         int32_t N, const void* target_logits, int64_t ld_t,
                                         float temperature, const void* draft, int64_t ld_q,
                                         const int32_t* draft_tokens, const int32_t* draft_len,
                                         const uint64_t* request_ids, uint32_t step,
                                         cosine_weight_mode_t weight_mode, int32_t* accept_len,
                                         int32_t* out_tokens, int32_t* status,
                                         const cosine_debug_t* debug) {
  cosine_status_t s = check_common(ctx, B, k, N);
  if (s != COSINE_OK) return s;
  if (ctx->cfg.nranks > 1)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "cosine_verify_batch_lazy runs on unsharded contexts (nranks == 1)");
  if (B == 0) { ctx->last_launches = 0; return COSINE_OK; }
  if ((s = check_rows(ctx, target_logits, ld_t, ctx->cfg.target_dtype, "target_logits")) != COSINE_OK) return s;
  if ((s = check_rows(ctx, draft, ld_q, ctx->cfg.draft_dtype, "draft")) != COSINE_OK) return s;
  if (!draft_tokens || !request_ids || !accept_len || !out_tokens || !status)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "NULL required pointer");
  if (!(temperature >= 0.f) || !std::isfinite(temperature))
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "temperature must be finite and >= 0");
  if ((int)weight_mode < 0 || (int)weight_mode > 3)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "bad weight mode");
  if (temperature == 0.f && ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "greedy (T = 0) needs PROBS drafts");
  DeviceGuard dg(ctx->cfg.device);
  Params P;
  fill_common(P, ctx, B, k, N, temperature);
  SplitParams S;
  memset(&S, 0, sizeof(S));
  S.B = B; S.k = k; S.N = N;
  S.V = P.V; S.ld_t = ld_t; S.ld_q = ld_q; S.ngroups = P.ngroups; S.gfull = P.gfull;
  S.k2f = P.k2f; S.k2d = P.k2d; S.greedy = P.greedy; S.weight_mode = weight_mode;
  S.target = target_logits; S.draft = draft; S.draft_tokens = draft_tokens; S.draft_len = draft_len;
  S.rids = request_ids; S.seed = P.seed; S.step = step;
  S.accept_len = accept_len; S.out_tokens = out_tokens; S.status = status;
  if (debug) S.dbg = *debug;
  return launch_lazy(ctx, (cudaStream_t)stream, S, ctx->cfg.target_dtype, ctx->cfg.draft_dtype,
                     ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS);
}

static cosine_status_t verify_tree_impl(bool lazy, cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t J,
                                   int32_t I, int32_t N, const int32_t* parent,
                                   const int32_t* node_token, const int32_t* internal_row,
                                   const void* target, int64_t ld_t, float temperature,
                                   const void* draft, int64_t ld_q,
                                   const int32_t* node_draft_tokens, const uint64_t* request_ids,
                                   uint32_t step, cosine_weight_mode_t weight_mode,
                                   int32_t* accept_len, int32_t* accepted_nodes,
                                   int32_t* out_tokens, int32_t* status) {
  cosine_status_t s = check_common(ctx, B, 1, N);
  if (s != COSINE_OK) return s;
  if (ctx->cfg.nranks > 1)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "cosine_verify_tree runs on unsharded contexts (nranks == 1)");
  if (J < 0 || J + 1 > ctx->cfg.max_tree_nodes)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "J + 1 exceeds max_tree_nodes");
  if (I < 0 || I > J + 1) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "I outside [0, J + 1]");
  if (B == 0) { ctx->last_launches = 0; return COSINE_OK; }
  if ((s = check_rows(ctx, target, ld_t, ctx->cfg.target_dtype, "target")) != COSINE_OK) return s;
  if (I > 0 && (s = check_rows(ctx, draft, ld_q, ctx->cfg.draft_dtype, "draft")) != COSINE_OK) return s;
  if (!parent || !node_token || !internal_row || (I > 0 && !node_draft_tokens) || !request_ids ||
      !accept_len || !accepted_nodes || !out_tokens || !status)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "NULL required pointer");
  if (!(temperature > 0.f) || !std::isfinite(temperature))
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "tree verification needs a finite temperature > 0");
  if ((int)weight_mode < 0 || (int)weight_mode > 2)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "tree weight mode must be CONF, WINNER or UNIFORM");
  const int64_t ngroups = (ctx->V + kGroup - 1) / kGroup;
  const int nmax = N <= 4 ? 4 : 8;
  const int esz = (int)std::max(esize(ctx->cfg.target_dtype), esize(ctx->cfg.draft_dtype));
  const int tg = tree_tile_groups(nmax, esz);
  if ((ngroups + tg - 1) / tg > kMaxSeg)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "vocabulary too wide for the tree sampler");
  DeviceGuard dg(ctx->cfg.device);
  Params P0;
  fill_common(P0, ctx, B, 1, N, temperature);
  TreeParams T;
  memset(&T, 0, sizeof(T));
  SplitParams& S = T.S;
  S.B = B; S.k = 1; S.N = N;
  S.V = P0.V; S.ld_t = ld_t; S.ld_q = ld_q; S.ngroups = P0.ngroups; S.gfull = P0.gfull;
  S.k2f = P0.k2f; S.k2d = P0.k2d; S.greedy = 0; S.weight_mode = weight_mode;
  S.target = target; S.draft = draft; S.rids = request_ids; S.seed = P0.seed; S.step = step;
  S.accept_len = accept_len; S.out_tokens = out_tokens; S.status = status;
  S.tree = 1; S.nn = J + 1; S.I = I; S.irow = internal_row;
  S.parts = ctx->parts;
  T.parent = parent; T.node_token = node_token; T.node_draft_tokens = node_draft_tokens;
  T.ndec = ctx->ndec; T.cpq = ctx->cpq; T.accepted_nodes = accepted_nodes;
  T.lazy = lazy ? 1 : 0;
  const int64_t units = (int64_t)B * (J + 1);
  int C = 1;
  if (ctx->cfg.cluster_size > 0) {
    C = ctx->cfg.cluster_size;
  } else {
    while (C < kMaxC && S.ngroups > (int64_t)C * kThreads * 8) C *= 2;
    while (C < kMaxC && units * C < 148 * 8 && S.ngroups >= (int64_t)C * 2 * kThreads) C *= 2;
  }
  S.C = C;
  S.cg = (S.ngroups + C - 1) / C;
  SplitFn sf[3];
  pick_split(ctx->cfg.target_dtype, ctx->cfg.draft_dtype, ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS, N, sf);
  TreeFn tf[2];
  pick_tree(ctx->cfg.target_dtype, ctx->cfg.draft_dtype, ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS, N, tf);
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaError_t e = cudaSuccess;
  if (!lazy) {
    lc.gridDim = dim3((unsigned)(units * C), 1, 1);
    e = cudaLaunchKernelEx(&lc, sf[0], S);  // every node's rows, once
    if (e == cudaSuccess) {
      lc.gridDim = dim3((unsigned)((units + kWarps - 1) / kWarps), 1, 1);
      lc.attrs = at;
      lc.numAttrs = 1;
      e = cudaLaunchKernelEx(&lc, tf[0], T);
    }
  }
  if (e == cudaSuccess) {
    lc.gridDim = dim3((unsigned)B, 1, 1);
    lc.blockDim = dim3(kTreeBlock, 1, 1);
    lc.dynamicSmemBytes = (size_t)tree_walk_smem(nmax, (ngroups + tg - 1) / tg);
    cudaFuncAttributes fa;
    int optin = 0;
    e = cudaFuncGetAttributes(&fa, tf[1]);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->cfg.device);
    if (e == cudaSuccess && fa.sharedSizeBytes + lc.dynamicSmemBytes > (size_t)optin) {
      ctx->last_launches = 2;
      return fail(ctx, COSINE_ERR_UNSUPPORTED, "vocabulary too wide for the tree walk's shared memory");
    }
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tf[1], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lc.dynamicSmemBytes);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&lc, tf[1], T);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("tree kernels: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = lazy ? 1 : 3;
  return COSINE_OK;
}

cosine_status_t cosine_verify_tree(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t J,
                                   int32_t I, int32_t N, const int32_t* parent,
                                   const int32_t* node_token, const int32_t* internal_row,
                                   const void* target, int64_t ld_t, float temperature,
                                   const void* draft, int64_t ld_q,
                                   const int32_t* node_draft_tokens, const uint64_t* request_ids,
                                   uint32_t step, cosine_weight_mode_t weight_mode,
                                   int32_t* accept_len, int32_t* accepted_nodes,
                                   int32_t* out_tokens, int32_t* status) {
  return verify_tree_impl(false, ctx, stream, B, J, I, N, parent, node_token, internal_row, target, ld_t,
                          temperature, draft, ld_q, node_draft_tokens, request_ids, step, weight_mode,
                          accept_len, accepted_nodes, out_tokens, status);
}

cosine_status_t cosine_fuse_step(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t N,
                                 const void* logits, int64_t ld, float temperature, int32_t* own_tokens,
                                 float* conf, int32_t* fused_token, int32_t* winner, int32_t* status) {
  cosine_status_t s = check_common(ctx, B, 1, N);
  if (s != COSINE_OK) return s;
  if (ctx->cfg.nranks > 1)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "cosine_fuse_step runs on unsharded contexts (nranks == 1)");
  if (B == 0) { ctx->last_launches = 0; return COSINE_OK; }
  if ((s = check_rows(ctx, logits, ld, ctx->cfg.draft_dtype, "logits")) != COSINE_OK) return s;
  if (!own_tokens || !conf || !fused_token || !winner || !status)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "NULL required pointer");
  if (!(temperature > 0.f) || !std::isfinite(temperature))
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "fuse_step needs a finite temperature > 0");
  DeviceGuard dg(ctx->cfg.device);
  FuseStepParams F;
  memset(&F, 0, sizeof(F));
  F.B = B; F.N = N; F.V = ctx->V; F.ld = ld;
  F.ngroups = (ctx->V + kGroup - 1) / kGroup;
  F.gfull = ctx->V / kGroup;
  F.k2f = (float)(1.4426950408889634 / (double)temperature);
  const int64_t rows = (int64_t)B * N;
  // one row per CTA (16 B per load): ~32 groups per thread keep the per-CTA reduction cheap
  int C = 1;
  while (C < kMaxC && F.ngroups > (int64_t)C * kThreads * 32) C *= 2;
  while (C < kMaxC && rows * C < 148 * 6 && F.ngroups >= (int64_t)C * 2 * kThreads) C *= 2;
  if (const char* v = getenv("COSINE_FUSE_STEP_C")) C = std::max(1, std::min(kMaxC, atoi(v)));
  while (C > 1 && (size_t)(rows * C) > ctx->parts_cap) C /= 2;
  if ((size_t)(rows * C) > ctx->parts_cap)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "B * N exceeds the context's scratch (raise max_batch / max_draft_len)");
  F.C = C;
  F.cg = (F.ngroups + C - 1) / C;
  F.logits = logits;
  F.parts = ctx->parts;
  F.own_tokens = own_tokens; F.conf = conf; F.fused_token = fused_token; F.winner = winner; F.status = status;
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.stream = (cudaStream_t)stream;
  lc.gridDim = dim3((unsigned)(rows * C), 1, 1);
  cudaError_t e = (ctx->cfg.draft_dtype == COSINE_BF16)
                      ? cudaLaunchKernelEx(&lc, fuse_step_stats_kernel<__nv_bfloat16>, F)
                      : cudaLaunchKernelEx(&lc, fuse_step_stats_kernel<float>, F);
  if (e == cudaSuccess) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    lc.gridDim = dim3((unsigned)((B + kWarps - 1) / kWarps), 1, 1);
    e = cudaLaunchKernelEx(&lc, fuse_step_combine_kernel, F);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("fuse_step kernels: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = 2;
  return COSINE_OK;
}

cosine_status_t cosine_route_update(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t N, int32_t K,
                                    const int32_t* draft_tokens, const float* conf, const int32_t* accepted,
                                    int64_t acc_stride, const int32_t* accept_len, const void* emb,
                                    int64_t hidden, int64_t ld_e, cosine_dtype_t emb_dtype,
                                    const uint8_t* participating, float decay, float* M, float* d_out,
                                    int32_t* status) {
  if (!ctx) return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "NULL context");
  if (B < 0 || B > ctx->cfg.max_batch) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "B outside [0, max_batch]");
  if (N < 1 || N > kWarps * 4 || K < 1 || acc_stride < K)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "bad N / K / acc_stride");
  if (B == 0) { ctx->last_launches = 0; return COSINE_OK; }
  if (!draft_tokens || !conf || !accepted || !accept_len || !emb || !M || !status)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "NULL required pointer");
  if (emb_dtype != COSINE_BF16 && emb_dtype != COSINE_F32)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "embedding dtype must be COSINE_BF16 or COSINE_F32");
  if (hidden < 8 || hidden % 8 != 0 || ld_e < hidden || !aligned16(emb) || ((uint64_t)ld_e * esize(emb_dtype)) % 16 != 0)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "embedding rows: hidden % 8 == 0, 16-byte aligned rows");
  if (!(decay >= 0.f && decay <= 1.f)) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "decay outside [0, 1]");
  DeviceGuard dg(ctx->cfg.device);
  RouteParams R;
  memset(&R, 0, sizeof(R));
  R.B = B; R.N = N; R.K = K; R.V = ctx->cfg.vocab_size; R.Hd = hidden; R.ld_e = ld_e; R.acc_stride = acc_stride;
  R.draft_tokens = draft_tokens; R.conf = conf; R.accepted = accepted; R.accept_len = accept_len; R.emb = emb;
  R.participating = participating; R.decay = decay; R.eps = 1e-6f; R.M = M; R.d_out = d_out; R.status = status;
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.gridDim = dim3((unsigned)B, 1, 1);
  lc.stream = (cudaStream_t)stream;
  cudaError_t e = (emb_dtype == COSINE_BF16) ? cudaLaunchKernelEx(&lc, route_update_kernel<__nv_bfloat16>, R)
                                             : cudaLaunchKernelEx(&lc, route_update_kernel<float>, R);
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("route_update: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = 1;
  return COSINE_OK;
}

cosine_status_t cosine_tree_select(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t S, int32_t K,
                                   const int32_t* tokens, const float* conf, int32_t budget, int32_t* n_nodes,
                                   int32_t* parent, int32_t* token, float* score, int32_t* depth) {
  if (!ctx) return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "NULL context");
  if (B < 0 || S < 1 || K < 1 || budget < 0 || (int64_t)S * K + 1 > kSelMaxNodes)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "bad B / S / K / budget (S * K + 1 <= 1024)");
  if (B == 0) { ctx->last_launches = 0; return COSINE_OK; }
  if (!tokens || !conf || !n_nodes || !parent || !token || !score || !depth)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "NULL required pointer");
  DeviceGuard dg(ctx->cfg.device);
  TreeSelParams T;
  memset(&T, 0, sizeof(T));
  T.B = B; T.S = S; T.K = K; T.budget = budget; T.tokens = tokens; T.conf = conf;
  T.n_nodes = n_nodes; T.parent = parent; T.token = token; T.score = score; T.depth = depth;
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.gridDim = dim3((unsigned)B, 1, 1);
  lc.stream = (cudaStream_t)stream;
  const cudaError_t e = cudaLaunchKernelEx(&lc, tree_select_kernel, T);
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("tree_select: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = 1;
  return COSINE_OK;
}

cosine_status_t cosine_verify_tree_lazy(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t J,
                                        int32_t I, int32_t N, const int32_t* parent,
                                        const int32_t* node_token, const int32_t* internal_row,
                                        const void* target, int64_t ld_t, float temperature,
                                        const void* draft, int64_t ld_q,
                                        const int32_t* node_draft_tokens, const uint64_t* request_ids,
                                        uint32_t step, cosine_weight_mode_t weight_mode,
                                        int32_t* accept_len, int32_t* accepted_nodes,
                                        int32_t* out_tokens, int32_t* status) {
  return verify_tree_impl(true, ctx, stream, B, J, I, N, parent, node_token, internal_row, target, ld_t,
                          temperature, draft, ld_q, node_draft_tokens, request_ids, step, weight_mode,
                          accept_len, accepted_nodes, out_tokens, status);
}

cosine_status_t cosine_sample_residual(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B,
                                       const void* target_rows, int64_t ld_t, float temperature,
                                       const float* row_max, const float* row_sumexp,
                                       const void* draft_rows, int64_t ld_q, const float* weights,
                                       const float* draft_norm, int32_t N,
                                       const uint32_t* node_ids, const uint64_t* request_ids,
                                       uint32_t step, int32_t* out_token, int32_t* status) {
  const int Nc = draft_rows ? N : 1;
  cosine_status_t s = check_common(ctx, B, 1, Nc);
  if (s != COSINE_OK) return s;
  if (ctx->cfg.nranks > 1)
    return fail(ctx, COSINE_ERR_UNSUPPORTED, "cosine_sample_residual runs on unsharded contexts (nranks == 1)");
  if (B == 0) { ctx->last_launches = 0; return COSINE_OK; }
  if ((s = check_rows(ctx, target_rows, ld_t, ctx->cfg.target_dtype, "target_rows")) != COSINE_OK) return s;
  if (draft_rows) {
    if ((s = check_rows(ctx, draft_rows, ld_q, ctx->cfg.draft_dtype, "draft_rows")) != COSINE_OK) return s;
    if (!weights || !draft_norm) return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "weights / draft_norm are NULL");
    if (ctx->cfg.draft_kind != COSINE_DRAFT_PROBS)
      return fail(ctx, COSINE_ERR_UNSUPPORTED, "sample_residual takes PROBS drafter rows");
  }
  if (!node_ids || !request_ids || !out_token || !status)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "NULL required pointer");
  if ((row_max == nullptr) != (row_sumexp == nullptr))
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "row_max and row_sumexp must both be given or both NULL");
  if (!(temperature >= 0.f) || !std::isfinite(temperature))
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "temperature must be finite and >= 0");
  DeviceGuard dg(ctx->cfg.device);
  Params P;
  fill_common(P, ctx, B, 1, Nc, temperature);
  P.mode = kModeSample;
  P.ld_t = ld_t;
  P.ld_q = ld_q;
  P.target = target_rows;
  P.draft = draft_rows;
  P.row_max = row_max;
  P.row_sumexp = row_sumexp;
  P.w_in = weights;
  P.norm_in = draft_norm;
  P.node_ids = node_ids;
  P.rids = request_ids;
  P.step = step;
  P.out_token = out_token;
  P.status = status;
  return launch(ctx, (cudaStream_t)stream, P, (int64_t)B, ctx->cfg.target_dtype,
                ctx->cfg.draft_dtype, false);
}

}  // extern "C"
