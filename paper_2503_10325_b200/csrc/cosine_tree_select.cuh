// cosine_tree_select.cuh — TreeSelection (Alg. 1 "TreeSelection" P:372,
// SPEC S:303-311 construction, reading #25): one CTA per request.
//   1. warp 0 merges the S branches into a prefix tree in shared memory (lane-parallel child
//      search); a node's score = the largest product of confidences along a branch reaching it;
//   2. every thread ranks its nodes (score desc, depth asc, creation order): the best `budget`
//      non-root nodes are kept (prefix-closed: scores never grow along a path);
//   3. breadth-first renumbering, depth by depth, siblings by (score desc, creation order), so the
//      output satisfies cosine_verify_tree's parent[j] < j / slot order.
#pragma once

#include "cosine_common.cuh"

namespace cosine {

constexpr int kSelMaxNodes = 1024;

struct TreeSelParams {
  int B, S, K, budget;
  const int32_t* tokens;  // [B][S][K]
  const float* conf;      // [B][S][K]
  int32_t* n_nodes;       // [B]
  int32_t* parent;        // [B][budget + 1]
  int32_t* token;         // [B][budget + 1]
  float* score;           // [B][budget + 1]
  int32_t* depth;         // [B][budget + 1]
};

__global__ void __launch_bounds__(kThreads) tree_select_kernel(const TreeSelParams P) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  __shared__ int32_t tp[kSelMaxNodes], tt[kSelMaxNodes], td[kSelMaxNodes], keep[kSelMaxNodes], nid[kSelMaxNodes];
  __shared__ double ts[kSelMaxNodes];
  __shared__ int s_n, s_base;
  const int S = P.S, K = P.K;
  if (warp == 0) {  // 1. prefix merge (sequential over the branches, lane-parallel search)
    int n = 1;
    if (lane == 0) { tp[0] = -1; tt[0] = -1; td[0] = 0; ts[0] = 1.0; }
    for (int s2 = 0; s2 < S; ++s2) {
      int cur = 0;
      double prod = 1.0;
      for (int i = 0; i < K; ++i) {
        const int32_t x = P.tokens[((int64_t)b * S + s2) * K + i];
        if (x < 0) break;
        prod *= (double)P.conf[((int64_t)b * S + s2) * K + i];
        __syncwarp();
        int child = -1;
        for (int c0 = 1; c0 < n && child < 0; c0 += 32) {
          const int c = c0 + lane;
          const unsigned m = __ballot_sync(0xffffffffu, c < n && tp[c] == cur && tt[c] == x);
          if (m) child = c0 + __ffs(m) - 1;
        }
        if (child < 0) {
          child = n++;
          if (lane == 0) { tp[child] = cur; tt[child] = x; td[child] = td[cur] + 1; ts[child] = prod; }
        } else if (lane == 0 && prod > ts[child]) {
          ts[child] = prod;
        }
        cur = child;
      }
    }
    if (lane == 0) s_n = n;
  }
  __syncthreads();
  const int n = s_n;
  // 2. keep the budget best non-root nodes
  for (int c = tid; c < n; c += kThreads) {
    int rank = 0;
    if (c > 0)
      for (int c2 = 1; c2 < n; ++c2)
        rank += (ts[c2] > ts[c] || (ts[c2] == ts[c] && (td[c2] < td[c] || (td[c2] == td[c] && c2 < c)))) ? 1 : 0;
    keep[c] = (c == 0) || rank < P.budget;
    nid[c] = (c == 0) ? 0 : -1;
  }
  if (tid == 0) s_base = 1;
  __syncthreads();
  // 3. breadth-first renumbering
  for (int d = 1; d <= K; ++d) {
    int cnt = 0;
    for (int c = tid; c < n; c += kThreads) {
      if (!keep[c] || td[c] != d) continue;
      int rank = 0;
      const int pc = nid[tp[c]];
      for (int c2 = 1; c2 < n; ++c2) {
        if (!keep[c2] || td[c2] != d) continue;
        const int pc2 = nid[tp[c2]];
        rank += (pc2 < pc || (pc2 == pc && (ts[c2] > ts[c] || (ts[c2] == ts[c] && c2 < c)))) ? 1 : 0;
      }
      nid[c] = s_base + rank;
      ++cnt;
    }
    __syncthreads();
    if (cnt) atomicAdd(&s_base, cnt);  // every thread read s_base before this barrier
    __syncthreads();
  }
  const int64_t o = (int64_t)b * (P.budget + 1);
  for (int j = tid; j <= P.budget; j += kThreads) {
    P.parent[o + j] = -1; P.token[o + j] = -1; P.score[o + j] = 0.f; P.depth[o + j] = -1;
  }
  __syncthreads();
  for (int c = tid; c < n; c += kThreads) {
    if (!keep[c]) continue;
    const int j = nid[c];
    P.parent[o + j] = (c == 0) ? -1 : nid[tp[c]];
    P.token[o + j] = tt[c];
    P.score[o + j] = (float)ts[c];
    P.depth[o + j] = td[c];
  }
  if (tid == 0) P.n_nodes[b] = s_base;
}

}  // namespace cosine
