// cosine_common.cuh — sampling-weight kinds, the Decision record and the block-wide
// inverse-CDF scan shared by the verification kernels (independent of the oracle).
#pragma once

#include "cosine_kernels.cuh"
#include "cosine_verify.h"

namespace cosine {

// Sampling weight kinds (what w(v) a sampling round draws from).
enum WKind : int {
  kWBonus = 0,     // exp((l - M)/T)
  kWResidual = 1,  // max(0, p - q), q = sum_n a_n d_n
  kWPoint = 2,     // max(0, p - delta_{x*})                    (POINT mode)
  kWFuseQ = 3,     // q (SAMPLE select: x* ~ q)                 (reading #3)
  kWProb = 4,      // p (degenerate residual fallback)    (reading #11)
  kWWriteQ = 5     // materialise q into fused_q (fuse_drafts)
};

struct Decision {
  int32_t need, kind, xstar;
  uint32_t node;
  double u;
  float M, invS, k2;
  float a[kMaxN], dm[kMaxN];
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
template <typename TT, typename TQ, bool kLogits, int NMAX, int kBar = 0, typename PP>
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

}  // namespace cosine
