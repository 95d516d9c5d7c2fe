// cosine_route.cuh — routing feedback after verification (Alg. 1 "Update
// routing matrix", Eq. 1, Eq. 2): one CTA per request, one warp per node.
//   d_{n,i} = cos(H(x_i), H(X_{n,i})) for i < L_b (embedding rows, lanes over the hidden dim,
//             128-bit loads, fp32 lane sums -> fp64 warp sums), else 0          (Eq. 1)
//   m_n = (1/K) sum_i c d / (c d + (1 - c)(1 - d)), c, d clamped to [eps, 1 - eps]   (Eq. 2)
// Non-participating nodes decay toward 0.5.  Tokens outside [0, V): status 2, M kept.
#pragma once

#include "cosine_common.cuh"

namespace cosine {

struct RouteParams {
  int B, N, K;
  int64_t V, Hd, ld_e, acc_stride;
  const int32_t* draft_tokens;  // [B][N][K]
  const float* conf;            // [B][N][K]
  const int32_t* accepted;      // [B][acc_stride]
  const int32_t* accept_len;    // [B]
  const void* emb;              // [V][ld_e]
  const uint8_t* participating; // [B][N] or NULL
  float decay, eps;
  float* M;                     // [B][N] in / out
  float* d_out;                 // [B][N][K] or NULL
  int32_t* status;              // [B]
};

template <typename T>
__global__ void __launch_bounds__(kThreads) route_update_kernel(const RouteParams P) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const int N = P.N, K = P.K;
  const int L = P.accept_len[b];
  __shared__ int s_bad;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  if (L >= 0) {  // every token the request's feedback touches must be a vocabulary row
    for (int j = tid; j < N * K; j += kThreads) {
      const int32_t x = P.draft_tokens[(int64_t)b * N * K + j];
      if (x < 0 || (int64_t)x >= P.V) atomicOr(&s_bad, 1);
    }
    for (int i = tid; i < K && i < L; i += kThreads) {
      const int32_t a = P.accepted[(int64_t)b * P.acc_stride + i];
      if (a < 0 || (int64_t)a >= P.V) atomicOr(&s_bad, 1);
    }
  }
  __syncthreads();
  if (tid == 0) P.status[b] = (L >= 0 && s_bad) ? COSINE_REQ_TOKEN_OUT_OF_RANGE : 0;
  if (L < 0 || s_bad) return;  // no feedback for a failed request / bad tokens
  const T* E = (const T*)P.emb;
  const int64_t ng = P.Hd / kGroup;  // 8-element groups per embedding row
  for (int n = warp; n < N; n += kWarps) {
    const int64_t bn = (int64_t)b * N + n;
    if (P.participating && !P.participating[bn]) {
      if (lane == 0) P.M[bn] = 0.5f + P.decay * (P.M[bn] - 0.5f);
      continue;
    }
    double m = 0.0;
    for (int i = 0; i < K; ++i) {
      double d = 0.0;
      if (i < L) {  // Eq. 1: cosine similarity of the accepted and the drafted token's embeddings
        const T* ea = E + (int64_t)P.accepted[(int64_t)b * P.acc_stride + i] * P.ld_e;
        const T* ex = E + (int64_t)P.draft_tokens[bn * K + i] * P.ld_e;
        float ab = 0.f, aa = 0.f, xx = 0.f;
        for (int64_t g = lane; g < ng; g += 32) {
          Group<T> ga, gx;
          ga.load(ea, g);
          gx.load(ex, g);
          float fa[8], fx[8];
          ga.unpack(fa);
          gx.unpack(fx);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            ab = fmaf(fa[e], fx[e], ab);
            aa = fmaf(fa[e], fa[e], aa);
            xx = fmaf(fx[e], fx[e], xx);
          }
        }
        const double dab = warp_sum((double)ab), daa = warp_sum((double)aa), dxx = warp_sum((double)xx);
        d = (daa > 0.0 && dxx > 0.0) ? dab / (sqrt(daa) * sqrt(dxx)) : 0.0;
      }
      if (P.d_out && lane == 0) P.d_out[bn * K + i] = (float)d;
      double c = (double)P.conf[bn * K + i];
      const double eps = (double)P.eps;
      c = c < eps ? eps : (c > 1.0 - eps ? 1.0 - eps : c);
      d = d < eps ? eps : (d > 1.0 - eps ? 1.0 - eps : d);
      m += c * d / (c * d + (1.0 - c) * (1.0 - d));  // Eq. 2
    }
    if (lane == 0) P.M[bn] = (float)(m / K);
  }
}

}  // namespace cosine
