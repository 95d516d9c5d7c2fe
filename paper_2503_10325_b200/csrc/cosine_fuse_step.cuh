// cosine_fuse_step.cuh — drafter-side token fusion of one drafting iteration (SURVEY §8(f)
// NEXT-2): Alg. 1 Fuse and Eq. 4's first line over the N drafters'
// LM-head outputs, greedy drafting.  Per drafter row: its own token X_n = argmax (lowest
// index on ties) and its probability c_n = softmax(l_n / T)(X_n) = 1 / sum_v 2^((l_n(v) - max) k2);
// then x* = X_{n*}, n* = argmax_n c_n (lowest n on ties).
//
//   fuse_step_stats_kernel: one CTA per (request, drafter, vocabulary chunk) streams its chunk
//     once (128-bit loads): running max + lowest-index argmax and the online sum-exp (the
//     stats_kernel scheme: 2^(l k2 - fl(m k2)), corrected exactly in fp64 at the reduction);
//     writes one partial record.
//   fuse_step_combine_kernel: one warp per request combines the chunks of its N rows (fixed-order
//     fp64) and fuses.
#pragma once

#include "cosine_common.cuh"

namespace cosine {

struct FuseStepParams {
  int B, N, C;
  int64_t V, ld, ngroups, gfull, cg;
  float k2f;
  const void* logits;  // [B][N][ld]
  PartRec* parts;      // [B][N][C]
  int32_t* own_tokens; // [B][N]
  float* conf;         // [B][N]
  int32_t* fused_token;// [B]
  int32_t* winner;     // [B]
  int32_t* status;     // [B]
};

template <typename T>
__global__ void __launch_bounds__(kThreads) fuse_step_stats_kernel(const FuseStepParams P) {
  const int C = P.C;
  const int64_t row = blockIdx.x / C;
  const int rank = (int)(blockIdx.x % C);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const T* r = (const T*)P.logits + row * P.ld;
  const float k2 = P.k2f;
  float bv = -INFINITY;  // running max (also the argmax value); sums are relative to fl(bv k2)
  int64_t bi = -1;
  float tmk = kNegBig, ts = 0.f;
  const int64_t gb = (int64_t)rank * P.cg, ge = min(P.ngroups, gb + P.cg), gfe = min(ge, P.gfull);
  // ~40 instructions per 8 elements: the index search and the rescale run only when the group
  // max improves; a NaN / +inf logit poisons the sum (detected at the combine)
  auto step = [&](const float (&f)[8], int64_t gi) {
    const float gm = max8(f);
    if (gm > bv) {  // ascending order: the first index of the new max wins ties
      int e0 = 0;
#pragma unroll
      for (int e = 7; e >= 0; --e)
        if (f[e] == gm) e0 = e;
      bi = gi * kGroup + e0;
      bv = gm;
      const float nmk = gm * k2;
      ts *= ex2(tmk - nmk);
      tmk = nmk;
    }
    float e8[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) e8[e] = ex2(fmaf(f[e], k2, -tmk));
    ts += sum8(e8);
  };
  // four groups of loads in flight per thread (one row per CTA: 16 B per load), processed in
  // ascending index order (the argmax keeps the first index on ties)
  constexpr int kU = 4;
  for (int64_t g0 = gb + tid; g0 < gfe; g0 += kU * kThreads) {
    Group<T> g[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (g0 + u * kThreads < gfe) g[u].load(r, g0 + u * kThreads);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (g0 + u * kThreads < gfe) {
        float f[8];
        g[u].unpack(f);
        step(f, g0 + u * kThreads);
      }
    }
  }
  if (gfe < ge && tid == (int)((gfe - gb) % kThreads)) {  // the row's partial last group
    float f[8];
    load_partial(r, gfe, P.V, -INFINITY, f);
    step(f, gfe);
  }
  __shared__ float s_v[kWarps];
  __shared__ int64_t s_i[kWarps];
  __shared__ double s_s[kWarps];
  float wv = bv;
  int64_t wi = bi;
  warp_argmax(wv, wi);
  if (lane == 0) { s_v[warp] = wv; s_i[warp] = wi; }
  __syncthreads();
  float Mc = -INFINITY;
  int64_t ix = -1;
  for (int w = 0; w < kWarps; ++w)
    if (s_i[w] >= 0 && (ix < 0 || s_v[w] > Mc || (s_v[w] == Mc && s_i[w] < ix))) { Mc = s_v[w]; ix = s_i[w]; }
  const float Mk = (ix >= 0) ? Mc : kNegBig;
  double tsd = (ts != 0.f) ? (double)ts * exp2((double)tmk - (double)Mk * (double)k2) : 0.0;
  tsd = warp_sum(tsd);
  if (lane == 0) s_s[warp] = tsd;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t += s_s[w];
    PartRec* rec = P.parts + row * C + rank;
    rec->tmax = Mk;   // chunk max (the sums are relative to it)
    rec->targ = ix;   // chunk argmax (global index), -1 if the chunk is all -inf
    rec->dmax[0] = Mc;
    rec->tsum = t;    // NaN / inf if the chunk has a NaN or +inf logit
    rec->bad = 0;
  }
}

__global__ void __launch_bounds__(kThreads) fuse_step_combine_kernel(const FuseStepParams P) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x * kWarps + warp;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the chunk records (PDL)
  if (b >= P.B) return;
  const int N = P.N, C = P.C;
  const double k2 = (double)P.k2f;
  int st = 0, nstar = -1;
  double cbest = -1.0;
  for (int n = 0; n < N; ++n) {
    const PartRec* pr = P.parts + ((int64_t)b * N + n) * C;
    const bool own = lane < C;
    float v = own ? pr[lane].dmax[0] : -INFINITY;
    int64_t ix = own ? pr[lane].targ : -1;
    warp_argmax(v, ix);  // X_n: best value, lowest index on ties
    const float tmax = own ? pr[lane].tmax : kNegBig;
    const float M = warp_max(tmax);
    const double ts = own ? pr[lane].tsum : 0.0;
    const double S = warp_sum(ts != 0.0 ? ts * exp2((double)tmax * k2 - (double)M * k2) : 0.0);
    int sn = 0;
    if (!isfinite(S) || (ix >= 0 && !isfinite(v))) sn = COSINE_REQ_NONFINITE_INPUT;  // NaN / +inf logit
    else if (ix < 0 || !(S > 0.0)) sn = COSINE_REQ_EMPTY_ROW;                        // all -inf
    if (!st && sn) st = sn;  // the first drafter row with an error decides the request
    const double c = sn ? NAN : 1.0 / S;  // P(X_n) = 2^0 / S
    if (lane == 0) {
      P.own_tokens[(int64_t)b * N + n] = sn ? -1 : (int32_t)ix;
      P.conf[(int64_t)b * N + n] = (float)c;
    }
    if (!sn && c > cbest) { cbest = c; nstar = n; }  // Eq. 4: the first most confident drafter
  }
  if (lane == 0) {
    P.status[b] = st;
    P.winner[b] = st ? -1 : nstar;
    P.fused_token[b] = st ? -1 : P.own_tokens[(int64_t)b * N + nstar];
    if (st)
      for (int n = 0; n < N; ++n) P.own_tokens[(int64_t)b * N + n] = -1;
  }
}

}  // namespace cosine
