// cosine_tree.cuh — tree-shaped drafts: multi-candidate
// recursive rejection over a draft tree ("merge them into a tree topology"),
// DESIGN.md reading #13: at node j the children are tested in slot order with
// u = U(rid, child, ACCEPT) against o_r(x) / q_r(x); on a rejection o_{r+1} = norm(max(0, o_r - q_r))
// (a full pass over node j's rows) and q_{r+1} = q_r without x, renormalised; when the children are
// exhausted y ~ o_r (U(rid, j, SAMPLE)); at a leaf y ~ o_j (the bonus).
//
// Kernels: the streaming stats_kernel in tree mode (every node's target row and, for internal
// nodes, its N drafter rows, read once) -> tree_decide_kernel (one warp per node: statistics,
// Eq. 4 fusion at the node, o_j(x_c) and q_j(x_c) of each child) -> tree_walk_kernel (one
// 1024-thread CTA per request: the sequential walk; full passes only on rejections and for the
// final draw).
#pragma once

#include "cosine_split.cuh"

namespace cosine {

struct NodeDec {  // per node (b, j)
  int32_t status;  // data error of the node (token > non-finite > empty > zero probability)
  float M, gap;    // max logit, Eq. 4 fusion margin (internal nodes)
  double S;
  float a[kMaxN], dm[kMaxN];  // w_n / sigma_n, drafter maxima (LOGITS)
};
struct ChildPQ {  // o_parent(x_c) and q_parent(x_c) of node c's token (before any rejection)
  double p, q;
};

struct TreeParams {
  SplitParams S;  // shapes, rows, stats scratch (tree mode)
  const int32_t* parent;       // [B][nn]
  const int32_t* node_token;   // [B][nn]
  const int32_t* node_draft_tokens;  // [B][I][N]
  NodeDec* ndec;               // [B][nn]
  ChildPQ* cpq;                // [B][nn]
  int32_t* accepted_nodes;     // [B][nn]
  int lazy;                    // NEXT-1: the walk computes the statistics of the nodes it visits
};

// ---------------- node decisions (one warp) ----------------
// The statistics of node j's rows, combined over the whole vocabulary (valid in every lane;
// drafter n's sigma_n and LOGITS row max in lane n).
struct NodeStats {
  float M;
  double S;
  double sig;  // lane n < N
  float dmx;   // lane n < N
  bool t_nf, t_empty, d_nf, d_empty;
};

// One warp decides node j of request b from its row statistics: Eq. 4 fusion at the node
// (reading #2) and o_j(x_c), q_j(x_c) of every child c, lane-parallel (lane n holds
// drafter n's sigma_n and confidence; lanes over the children).  Writes the node record *nd_out
// (lane n: drafter n's fields, lane 0 the scalars); the child values go to gcpq[c] (global) or
// scp[c] / scq[c] (shared).  s_*: per-warp shared scratch.  Shared by tree_decide_kernel and the
// lazy walk.  Ends with __syncwarp().
template <typename TT, typename TQ, bool kLogits>
__device__ __forceinline__ void node_decide_warp(const TreeParams& T, int b, int j, int ir, bool has_d,
                                                 const TT* trow, const TQ* drow, const NodeStats& ns,
                                                 float* s_gx, int32_t* s_tok, double* s_w, double* s_sig,
                                                 float* s_dmax, int* s_zero, NodeDec* nd_out, ChildPQ* gcpq,
                                                 double* scp, double* scq) {
  const SplitParams& P = T.S;
  const int lane = threadIdx.x & 31;
  const int nn = P.nn, N = P.N;
  const double k2 = (double)P.k2f;
  if (lane == 0) *s_zero = 0;
  if (has_d && lane < N * N) {  // d_m(X_n) for the confidences at this node
    const int n = lane % N, m = lane / N;
    const int32_t tk = T.node_draft_tokens[((int64_t)b * P.I + ir) * N + n];
    float v = 0.f;
    if (tk >= 0 && (int64_t)tk < P.V) v = load_one(drow + (int64_t)m * P.ld_q, tk);
    s_gx[m * kMaxN + n] = v;
    if (m == 0) s_tok[n] = tk;
  }
  __syncwarp();
  const bool dl = lane < N;  // this lane holds a drafter
  const double sig_l = ns.sig;
  const float dmx_l = ns.dmx;
  bool tok_bad = false;
  if (has_d) {
    const int32_t t = dl ? s_tok[lane] : 0;
    tok_bad = __any_sync(0xffffffffu, dl && (t < 0 || (int64_t)t >= P.V));
  }
  int stc = tok_bad ? COSINE_REQ_TOKEN_OUT_OF_RANGE
                    : ((ns.t_nf || ns.d_nf) ? COSINE_REQ_NONFINITE_INPUT
                                            : ((ns.t_empty || ns.d_empty) ? COSINE_REQ_EMPTY_ROW : 0));
  double c_l = 0.0;  // c_n = q_n(X_n) at this node
  if (!stc && has_d) {
    if (dl) {
      const double dv = (double)s_gx[lane * kMaxN + lane];
      c_l = kLogits ? exp2(dv * k2 - (double)dmx_l * k2) / sig_l : dv / sig_l;
    }
    if (__any_sync(0xffffffffu, dl && c_l == 0.0)) stc = COSINE_REQ_ZERO_PROB_DRAFT;
  }
  const bool ok_for_children = !stc && has_d;
  float gap = INFINITY;
  double w_l = 0.0;
  if (ok_for_children) {  // Eq. 4 fusion weights at the node (reading #2)
    double bc = dl ? c_l : -1.0;
    int bn = dl ? lane : 1 << 30;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const int on = __shfl_xor_sync(0xffffffffu, bn, o);
      if (oc > bc || (oc == bc && on < bn)) { bc = oc; bn = on; }
    }
    double second = (dl && lane != bn) ? c_l : -1.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) second = fmax(second, __shfl_xor_sync(0xffffffffu, second, o));
    gap = (N > 1) ? (float)((bc - second) / bc) : INFINITY;
    if (P.weight_mode == COSINE_W_CONF) {
      const double sc = warp_sum(dl ? c_l : 0.0);
      w_l = dl ? c_l / sc : 0.0;
    } else if (P.weight_mode == COSINE_W_UNIFORM) {
      w_l = dl ? 1.0 / (double)N : 0.0;
    } else {
      w_l = (lane == bn) ? 1.0 : 0.0;
    }
    if (dl) {
      s_w[lane] = w_l;
      s_sig[lane] = sig_l;
      s_dmax[lane] = dmx_l;
    }
  }
  __syncwarp();
  // o_j(x_c), q_j(x_c) of every child c of j (lane-parallel over candidate node ids)
  for (int c = j + 1 + lane; c < nn; c += 32) {
    if (T.parent[(int64_t)b * nn + c] != j) continue;
    const int32_t x = T.node_token[(int64_t)b * nn + c];
    double pp = 0.0, qq = 0.0;
    if (x >= 0 && (int64_t)x < P.V && ok_for_children) {
      pp = exp2((double)load_one(trow, x) * k2 - (double)ns.M * k2) / ns.S;
      for (int m = 0; m < N; ++m) {
        const double dv = (double)load_one(drow + (int64_t)m * P.ld_q, x);
        const double qm = kLogits ? exp2(dv * k2 - (double)s_dmax[m] * k2) / s_sig[m] : dv / s_sig[m];
        qq += s_w[m] * qm;
      }
      if (qq == 0.0) atomicOr(s_zero, 1);  // a child the fused q cannot draw
    }
    if (gcpq) {
      ChildPQ pq;
      pq.p = pp;
      pq.q = qq;
      gcpq[c] = pq;
    } else {
      scp[c] = pp;
      scq[c] = qq;
    }
  }
  __syncwarp();
  if (lane < kMaxN) {
    const bool mine = ok_for_children && dl;
    nd_out->a[lane] = mine ? (float)(w_l / sig_l) : 0.f;
    nd_out->dm[lane] = mine ? dmx_l : 0.f;
  }
  if (lane == 0) {
    if (!stc && *s_zero) stc = COSINE_REQ_ZERO_PROB_DRAFT;
    nd_out->status = stc;
    nd_out->M = ns.M;
    nd_out->S = ns.S;
    nd_out->gap = gap;
  }
  __syncwarp();
}

// ---------------- kernel T1: one warp per node ----------------
template <typename TT, typename TQ, bool kLogits>
__global__ void __launch_bounds__(kThreads) tree_decide_kernel(const TreeParams T) {
  const SplitParams& P = T.S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t unit = (int64_t)blockIdx.x * kWarps + warp;
  __shared__ float s_gx[kWarps][kMaxN * kMaxN];
  __shared__ int32_t s_tok[kWarps][kMaxN];
  __shared__ double s_w[kWarps][kMaxN], s_sig[kWarps][kMaxN];
  __shared__ float s_dmax[kWarps][kMaxN];
  __shared__ int s_zero[kWarps];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the stats kernel's partial records (PDL)
  if (unit >= (int64_t)P.B * T.S.nn) return;
  const int nn = P.nn, N = P.N, C = P.C;
  const int b = (int)(unit / nn), j = (int)(unit % nn);
  const int ir = P.irow[unit];
  const bool has_d = ir >= 0 && ir < P.I;
  const double k2 = (double)P.k2f;
  const TT* trow = (const TT*)P.target + unit * P.ld_t;
  const TQ* drow = (const TQ*)P.draft + ((int64_t)b * P.I + (has_d ? ir : 0)) * N * P.ld_q;
  // combine the partial records (chunk r in lane r)
  const PartRec* parts = P.parts + unit * C;
  const bool own = lane < C;
  const float tmax = own ? parts[lane].tmax : kNegBig;
  const int bad = __reduce_or_sync(0xffffffffu, own ? parts[lane].bad : 0);
  NodeStats ns;
  ns.sig = NAN;
  ns.dmx = kNegBig;
  ns.M = warp_max(tmax);
  const double tsum = own ? parts[lane].tsum : 0.0;
  ns.S = warp_sum(tsum != 0.0 ? tsum * exp2((double)tmax * k2 - (double)ns.M * k2) : 0.0);
  ns.t_nf = !isfinite(ns.S) || !isfinite(ns.M);
  ns.t_empty = !ns.t_nf && !(ns.S > 0.0);
  ns.d_nf = false;
  ns.d_empty = false;
  if (has_d) {
    if (bad & 2) ns.d_nf = true;
    for (int n = 0; n < N; ++n) {
      double sv;
      float mx = kNegBig;
      const double ds = own ? parts[lane].dsum[n] : 0.0;
      if (kLogits) {
        const float dmr = own ? parts[lane].dmax[n] : kNegBig;
        mx = warp_max(dmr);
        sv = warp_sum(ds != 0.0 ? ds * exp2((double)dmr * k2 - (double)mx * k2) : 0.0);
        if (!isfinite(mx)) ns.d_nf = true;
      } else {
        sv = warp_sum(ds);
      }
      if (lane == n) { ns.sig = sv; ns.dmx = mx; }
      if (!isfinite(sv)) ns.d_nf = true;
      else if (!(sv > 0.0)) ns.d_empty = true;
    }
  }
  node_decide_warp<TT, TQ, kLogits>(T, b, j, ir, has_d, trow, drow, ns, s_gx[warp], s_tok[warp], s_w[warp],
                                    s_sig[warp], s_dmax[warp], &s_zero[warp], &T.ndec[unit],
                                    T.cpq + (int64_t)b * nn, nullptr, nullptr);
}

// ---------------- the walk ----------------
// One CTA per request: 16 consumer warps + 1 producer warp.  A full pass over node j's rows
// (target + N drafters) streams them through a kTreeStages-deep ring of shared-memory tiles filled
// by bulk async copies (TMA, cp.async.bulk) issued by the producer warp; full/empty mbarriers hand
// the stages over, so one SM keeps ~160 KB in flight without spending registers on it and the
// consumers never meet at a block barrier inside a pass.  Per-tile masses are kept for the final
// draw.
constexpr int kTreeWarps = 16;                      // consumer warps
constexpr int kTreeThreads = kTreeWarps * 32;       // consumer threads
constexpr int kTreeBlock = kTreeThreads + 32;       // + the producer warp
constexpr int kTreeMaxRej = 64;
constexpr int kTreeMaxNodes = 1024;  // nodes per tree (the walk stages the tree in shared memory)
// Ring geometry (measured on c4 with the latency trace, tools/tiny_trace.py walk): a pass is
// bound by the per-tile hand-over (consumer ~0.7 us per tile whatever its size) and the TMA
// turnaround under load (~2.9 us), so few large stages win: 2 x 80 KB tiles 27 us per pass
// (c4 1.405 ms, lazy 0.320 ms) vs 4 x 40 KB 29.5 us (1.423 / 0.350 ms), 8 x 20 KB 46 us,
// 3 x 60 KB (1.405 / 0.350 ms).
constexpr int kTreeStages = 2;

// Tile geometry: one tile = kTG groups of every row of the node; a row's slice is <= kRowB bytes.
__host__ __device__ constexpr int tree_row_bytes(int nmax) { return nmax <= 4 ? 16384 : 8192; }
__host__ __device__ constexpr int tree_tile_groups(int nmax, int esize_max) {
  return tree_row_bytes(nmax) / (kGroup * esize_max);
}
// Dynamic shared memory of the walk: the ring, then per-(tile, warp) partial masses.
__host__ __device__ constexpr int tree_walk_smem(int nmax, int64_t ntile) {
  return kTreeStages * (1 + nmax) * tree_row_bytes(nmax) + (int)ntile * kTreeWarps * 8;
}

struct TreeState {  // the current node's o_r, q_r as a recursion over r rejections
  float M, invS, k2;
  float a[kMaxN], dm[kMaxN];
  int r;
  int32_t xs[kTreeMaxRej];   // rejected tokens, in order
  double Zs[kTreeMaxRej];    // residual masses (0 = degenerate: o kept, reading #11)
  float invZ[kTreeMaxRej];   // 1 / Z (0 when degenerate)
  float qsc[kTreeMaxRej];    // 1 / (1 - q_t(x_t))
};

// The 8 weights of local group g of a staged tile, after rr recursion steps: mode 0 ->
// max(0, o_rr - q_rr) (the unnormalised residual, whose mass is Z_{rr+1}); mode 1 -> o_rr.
template <typename TT, typename TQ, bool kLogits, int NMAX>
__device__ __forceinline__ void tree_weights_s(const TreeState& st, int mode, int rr,
                                               const unsigned char* stage, int Nd, int g,
                                               int vbase, int V, float w[8]) {
  constexpr int kRowB = tree_row_bytes(NMAX);
  float t[8], q[8];
  Group<TT> tv;
  tv.load_s(reinterpret_cast<const TT*>(stage), g);
  tv.unpack(t);
#pragma unroll
  for (int e = 0; e < 8; ++e) q[e] = 0.f;
#pragma unroll
  for (int n = 0; n < NMAX; ++n) {
    if (n < Nd) {
      Group<TQ> dv;
      dv.load_s(reinterpret_cast<const TQ*>(stage + (1 + n) * kRowB), g);
      float f[8];
      dv.unpack(f);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float qv = kLogits ? ex2((f[e] - st.dm[n]) * st.k2) : f[e];
        q[e] = fmaf(st.a[n], qv, q[e]);
      }
    }
  }
  float pv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) pv[e] = ex2((t[e] - st.M) * st.k2) * st.invS;
  for (int s2 = 0; s2 < rr; ++s2) {
    const float iz = st.invZ[s2], qs = st.qsc[s2];
    const int xr = st.xs[s2] - vbase;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (iz > 0.f) pv[e] = fmaxf(pv[e] - q[e], 0.f) * iz;
      q[e] = (e == xr) ? 0.f : q[e] * qs;
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float x = (mode == 1) ? pv[e] : fmaxf(pv[e] - q[e], 0.f);
    w[e] = (vbase + e < V) ? x : 0.f;
  }
}

// Sum of the per-tile masses in a fixed order (one warp): lane l adds tiles l, l + 32, ...
__device__ __forceinline__ double tile_total(const double* s_tile, int64_t ntile, int lane) {
  double z = 0.0;
  for (int64_t t = lane; t < ntile; t += 32) z += s_tile[t];
  return warp_sum(z);
}

// Block barrier of the consumer warps only (named barrier 1; the producer warp is elsewhere).
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kTreeThreads) : "memory");
}

template <typename TT, typename TQ, int NMAX>
struct TreeRing {  // the shared-memory tile ring of one CTA
  static constexpr int kRowB = tree_row_bytes(NMAX);
  static constexpr int kEsz = sizeof(TT) > sizeof(TQ) ? (int)sizeof(TT) : (int)sizeof(TQ);
  static constexpr int kTG = tree_tile_groups(NMAX, kEsz);
  static constexpr int kStageB = (1 + NMAX) * kRowB;
  unsigned char* base;
  uint64_t* full;   // count 1: the producer's expect_tx arrival + the copies' bytes
  uint64_t* empty;  // count kTreeWarps: every consumer warp released the stage
  // Producer lane: fill ring slot `pos` (stage pos % S, its (pos / S)-th use) with tile `t` of
  // the node's rows (bytes up to V, rounded to 16), once the consumers released the previous use.
  __device__ __forceinline__ void fill(uint32_t pos, int64_t t, const SplitParams& P, const TT* trow,
                                       const TQ* drow, int Nd) const {
    const int stg = (int)(pos % kTreeStages);
    const uint32_t use = pos / kTreeStages;
    if (use > 0) mbar_wait_parity(&empty[stg], (use - 1) & 1u);
    fence_proxy_async_smem();
    const int64_t g0 = t * kTG;
    const int64_t e0 = g0 * kGroup, e1 = min((int64_t)P.V, (g0 + kTG) * kGroup);
    const uint32_t bt = (uint32_t)((((e1 - e0) * (int64_t)sizeof(TT)) + 15) & ~(int64_t)15);
    const uint32_t bq = (uint32_t)((((e1 - e0) * (int64_t)sizeof(TQ)) + 15) & ~(int64_t)15);
    unsigned char* dst = base + stg * kStageB;
    mbar_expect_tx(&full[stg], bt + (uint32_t)Nd * bq);
    bulk_g2s(dst, trow + e0, bt, &full[stg]);
    for (int n = 0; n < Nd; ++n) bulk_g2s(dst + (1 + n) * kRowB, drow + (int64_t)n * P.ld_q + e0, bq, &full[stg]);
  }
};

// Lazy walk (NEXT-1): the statistics of node j's rows, computed by the walk CTA itself when it
// arrives at j — one pass through the TMA ring (online max / sum-exp of the target row as in
// stats_kernel, drafter sums or online softmax statistics), a fixed-order block reduction, then
// warp 0 decides the node (node_decide_warp).  `it` (the ring position) advances by ntile.
template <typename TT, typename TQ, bool kLogits, int NMAX>
__device__ __forceinline__ void tree_node_stats(
    const TreeParams& T, int b, int j, int Nd, const TT* trow, const TQ* drow,
    const TreeRing<TT, TQ, NMAX>& ring, uint64_t* s_full, uint64_t* s_empty, uint32_t& it, int64_t ntile,
    bool producer, float (*s_rf)[1 + kMaxN], double (*s_rd)[1 + kMaxN], int* s_rbad, float* s_ngx,
    int32_t* s_ntok, double* s_nw, double* s_nsig, float* s_ndmax, int* s_nzero, NodeDec* s_nd, double* s_cp,
    double* s_cq, int ir) {
  using Ring = TreeRing<TT, TQ, NMAX>;
  constexpr int kTG = Ring::kTG;
  const SplitParams& P = T.S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float k2 = P.k2f;
  float tmx = kNegBig, tmk = kNegBig, ts = 0.f;
  float dm[NMAX], dmk[NMAX], ds[NMAX];
#pragma unroll
  for (int n = 0; n < NMAX; ++n) { dm[n] = kNegBig; dmk[n] = kNegBig; ds[n] = 0.f; }
  bool dneg = false;
  if (producer) {
    if (lane == 0)
      for (int64_t t = 0; t < ntile; ++t) ring.fill(it + (uint32_t)t, t, P, trow, drow, Nd);
  } else {
    for (int64_t t = 0; t < ntile; ++t) {
      const uint32_t pos = it + (uint32_t)t;
      const int stg = (int)(pos % kTreeStages);
      mbar_wait_parity(&s_full[stg], (pos / kTreeStages) & 1u);
      const unsigned char* sb = ring.base + stg * Ring::kStageB;
      const int64_t g0 = t * kTG;
      const int tg = (int)min((int64_t)kTG, P.ngroups - g0);
      for (int g = tid; g < tg; g += kTreeThreads) {
        const int vb = (int)((g0 + g) * kGroup);
        float f[8];
        Group<TT> tv;
        tv.load_s(reinterpret_cast<const TT*>(sb), g);
        tv.unpack(f);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (vb + e >= P.V) f[e] = -INFINITY;
        const float gm = max8(f);
        if (gm > tmx) {  // rescale by 2^(old fl(m k2) - new fl(m k2)); exact in fp64 below
          const float nmk = gm * k2;
          ts *= ex2(tmk - nmk);
          tmx = gm;
          tmk = nmk;
        }
        float e8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) e8[e] = ex2(fmaf(f[e], k2, -tmk));
        ts += sum8(e8);
#pragma unroll
        for (int n = 0; n < NMAX; ++n) {
          if (n < Nd) {
            Group<TQ> dv;
            dv.load_s(reinterpret_cast<const TQ*>(sb + (1 + n) * Ring::kRowB), g);
            dv.unpack(f);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (vb + e >= P.V) f[e] = kLogits ? -INFINITY : 0.f;
            if (kLogits) {
              const float dg = max8(f);
              if (dg > dm[n]) {
                const float nmk = dg * k2;
                ds[n] *= ex2(dmk[n] - nmk);
                dm[n] = dg;
                dmk[n] = nmk;
              }
#pragma unroll
              for (int e = 0; e < 8; ++e) e8[e] = ex2(fmaf(f[e], k2, -dmk[n]));
              ds[n] += sum8(e8);
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) dneg |= (f[e] < 0.f);
              ds[n] += sum8(f);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[stg]);
    }
  }
  it += (uint32_t)ntile;
  // fixed-order block reduction (consumer warps): maxima, then the sums rescaled in fp64
  if (!producer) {
    const float wm = warp_max(tmx);
    if (lane == 0) s_rf[warp][0] = wm;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      const float w = (kLogits && n < Nd) ? warp_max(dm[n]) : kNegBig;
      if (lane == 0) s_rf[warp][1 + n] = w;
    }
  }
  __syncthreads();
  if (!producer) {
    float Mc = kNegBig;
    for (int w2 = 0; w2 < kTreeWarps; ++w2) Mc = fmaxf(Mc, s_rf[w2][0]);
    double tsd = (ts != 0.f) ? (double)ts * exp2((double)tmk - (double)Mc * (double)k2) : 0.0;
    tsd = warp_sum(tsd);
    if (lane == 0) s_rd[warp][0] = tsd;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      if (n < Nd) {
        double dsd;
        if (kLogits) {
          float dMc = kNegBig;
          for (int w2 = 0; w2 < kTreeWarps; ++w2) dMc = fmaxf(dMc, s_rf[w2][1 + n]);
          dsd = (ds[n] != 0.f) ? (double)ds[n] * exp2((double)dmk[n] - (double)dMc * (double)k2) : 0.0;
        } else {
          dsd = (double)ds[n];
        }
        dsd = warp_sum(dsd);
        if (lane == 0) s_rd[warp][1 + n] = dsd;
      }
    }
    const int bad = __any_sync(0xffffffffu, dneg) ? 2 : 0;
    if (lane == 0) s_rbad[warp] = bad;
  }
  __syncthreads();
  if (warp == 0) {
    NodeStats ns;
    ns.sig = NAN;
    ns.dmx = kNegBig;
    float M = kNegBig;
    double S = 0.0;
    int bad = 0;
    for (int w2 = 0; w2 < kTreeWarps; ++w2) {
      M = fmaxf(M, s_rf[w2][0]);
      S += s_rd[w2][0];
      bad |= s_rbad[w2];
    }
    ns.M = M;
    ns.S = S;
    ns.t_nf = !isfinite(S) || !isfinite(M);
    ns.t_empty = !ns.t_nf && !(S > 0.0);
    ns.d_nf = (bad & 2) != 0;
    ns.d_empty = false;
    for (int n = 0; n < P.N; ++n) {
      double sv = 0.0;
      float mx = kNegBig;
      if (n < Nd) {
        for (int w2 = 0; w2 < kTreeWarps; ++w2) {
          sv += s_rd[w2][1 + n];
          if (kLogits) mx = fmaxf(mx, s_rf[w2][1 + n]);
        }
        if (kLogits && !isfinite(mx)) ns.d_nf = true;
        if (!isfinite(sv)) ns.d_nf = true;
        else if (!(sv > 0.0)) ns.d_empty = true;
      }
      if (lane == n) { ns.sig = sv; ns.dmx = mx; }
    }
    node_decide_warp<TT, TQ, kLogits>(T, b, j, ir, Nd > 0, trow, drow, ns, s_ngx, s_ntok, s_nw, s_nsig, s_ndmax,
                                      s_nzero, s_nd, nullptr, s_cp, s_cq);
  }
  __syncthreads();
}

template <typename TT, typename TQ, bool kLogits, int NMAX>
__global__ void __launch_bounds__(kTreeBlock, 1) tree_walk_kernel(const TreeParams T) {
  using Ring = TreeRing<TT, TQ, NMAX>;
  constexpr int kTG = Ring::kTG;
  const SplitParams& P = T.S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const int nn = P.nn, N = P.N;
  extern __shared__ __align__(128) unsigned char tree_smem[];
  __shared__ __align__(8) uint64_t s_full[kTreeStages], s_empty[kTreeStages];
  __shared__ TreeState st;
  __shared__ int s_act, s_node, s_Nd;
  __shared__ double s_tile[kMaxSeg];
  __shared__ double s_u;
  __shared__ int64_t s_y;
  __shared__ float s_margin;
  __shared__ int32_t par[kTreeMaxNodes], tok[kTreeMaxNodes], irw[kTreeMaxNodes];
  __shared__ int32_t s_e12[kTreeMaxNodes], s_e3[kTreeMaxNodes];  // structure (e1 | e2 << 8), data
  __shared__ double s_cp[kTreeMaxNodes], s_cq[kTreeMaxNodes];
  // lazy mode: the visited node's record and its statistics-pass scratch
  __shared__ NodeDec s_nd;
  __shared__ float s_rf[kTreeWarps][1 + kMaxN];
  __shared__ double s_rd[kTreeWarps][1 + kMaxN];
  __shared__ int s_rbad[kTreeWarps];
  __shared__ float s_ngx[kMaxN * kMaxN];
  __shared__ int32_t s_ntok[kMaxN];
  __shared__ double s_nw[kMaxN], s_nsig[kMaxN];
  __shared__ float s_ndmax[kMaxN];
  __shared__ int s_nzero, s_have, s_err;
  const Ring ring{tree_smem, s_full, s_empty};
  double* s_parts = reinterpret_cast<double*>(tree_smem + kTreeStages * Ring::kStageB);  // [ntile][warps]
  const bool producer = warp == kTreeWarps;
  if (tid == 0) {
    for (int i = 0; i < kTreeStages; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], kTreeWarps);
    }
    fence_mbar_init_cluster();
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // tree_decide_kernel's records (PDL)
  const NodeDec* nds = T.ndec + (int64_t)b * nn;
  const ChildPQ* cpq = T.cpq + (int64_t)b * nn;
  for (int c = tid; c < nn; c += kTreeBlock) {  // the tree and its per-node records, staged
    par[c] = T.parent[(int64_t)b * nn + c];
    tok[c] = T.node_token[(int64_t)b * nn + c];
    irw[c] = P.irow[(int64_t)b * nn + c];
    if (!T.lazy) {
      s_e3[c] = nds[c].status;
      s_cp[c] = cpq[c].p;
      s_cq[c] = cpq[c].q;
    } else {
      s_e3[c] = 0;  // lazy: a node's data errors are found when the walk visits it
    }
  }
  __syncthreads();
  int32_t* out = P.out_tokens + (int64_t)b * nn;
  int32_t* acc = T.accepted_nodes + (int64_t)b * nn;
  const uint64_t rid = P.rids[b];
  // structure checks, one node per thread: (1) parent order, token range, distinct siblings;
  // (2) internal rows exactly for the nodes with children; then (3) node data errors — the
  // first error in that order wins (reading #12, #13; same order as the oracle)
  for (int c = tid; c < nn; c += kTreeBlock) {
    int e1 = 0, e2 = 0;
    if (c == 0) {
      if (par[0] != -1) e1 = COSINE_REQ_BAD_TREE;
    } else if (par[c] < 0 || par[c] >= c) {
      e1 = COSINE_REQ_BAD_TREE;
    } else if (tok[c] < 0 || (int64_t)tok[c] >= P.V) {
      e1 = COSINE_REQ_TOKEN_OUT_OF_RANGE;
    } else {
      for (int c2 = 1; c2 < c; ++c2)
        if (par[c2] == par[c] && tok[c2] == tok[c]) { e1 = COSINE_REQ_BAD_TREE; break; }
    }
    bool has_child = false;
    for (int c2 = c + 1; c2 < nn; ++c2)
      if (par[c2] == c) { has_child = true; break; }
    if (has_child != (irw[c] >= 0) || irw[c] >= P.I) e2 = COSINE_REQ_BAD_TREE;
    s_e12[c] = e1 | (e2 << 8);
  }
  __syncthreads();
  // thread-0 walk state
  int err = 0, j = 0, depth = 0, ci = 0, deg = 0;
  float tm = INFINITY;
  bool need_init = true;
  if (tid == 0) {
    s_have = -1;
    for (int c = 0; c < nn && !err; ++c) err = s_e12[c] & 0xff;
    for (int c = 0; c < nn && !err; ++c) err = s_e12[c] >> 8;
    for (int c = 0; c < nn && !err; ++c) err = s_e3[c];
    s_act = err ? 0 : -1;
  }
  __syncthreads();
  if (s_act == 0) {
    for (int c = tid; c < nn; c += kTreeBlock) { out[c] = -1; acc[c] = -1; }
    if (tid == 0) { P.accept_len[b] = -1; P.status[b] = err; }
    return;
  }
  const int64_t ntile = (P.ngroups + kTG - 1) / kTG;
  uint32_t it = 0;  // tiles consumed so far (ring position and mbarrier phase), uniform
#ifdef COSINE_TRACE  // thread 0: time in the walk logic and in each kind of block step
  unsigned long long tr_prev = 0, tr_acc[5] = {0, 0, 0, 0, 0}, tr_cnt[5] = {0, 0, 0, 0, 0};
  int tr_act = -1;
  auto tr_now = []() { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); return t_; };
  if (tid == 0) {
    tr_prev = tr_now();
    if (P.trace) P.trace[(size_t)blockIdx.x * 16 + 0] = tr_prev;
  }
  auto tr_flush = [&]() {
    if (tid == 0 && P.trace) {
      const unsigned long long t = tr_now();
      if (tr_act >= 0) tr_acc[tr_act] += t - tr_prev;
      unsigned long long* o = P.trace + (size_t)blockIdx.x * 16;
      o[1] = t;
      for (int q = 0; q < 5; ++q) { o[2 + q] = tr_acc[q]; o[7 + q] = tr_cnt[q]; }
    }
  };
#endif
  for (;;) {
#ifdef COSINE_TRACE
    if (tid == 0) {  // the previous step's block work ends here
      const unsigned long long t = tr_now();
      if (tr_act >= 0) tr_acc[tr_act] += t - tr_prev;
      tr_prev = t;
    }
#endif
    if (tid == 0) {
      // advance the walk until the block is needed for a pass (act 1) or the final draw (act 2)
      int act = -1;
      while (act < 0) {
        if (need_init && T.lazy && s_have != j) {  // lazy: node j's statistics first (act 3)
          act = 3;
          break;
        }
        if (need_init) {  // arriving at node j: o_0, q_0 of the node
          const NodeDec& nd = T.lazy ? s_nd : nds[j];
          if (nd.status) {  // lazy: a data error of a visited node stops the request
            err = nd.status;
            act = 4;
            break;
          }
          st.M = nd.M;
          st.invS = (float)(1.0 / nd.S);
          st.k2 = P.k2f;
          for (int n = 0; n < kMaxN; ++n) { st.a[n] = nd.a[n]; st.dm[n] = nd.dm[n]; }
          st.r = 0;
          ci = j + 1;
          need_init = false;
          if (irw[j] >= 0 && P.weight_mode == COSINE_W_WINNER) tm = fmin_(tm, nd.gap);  // reading #18
        }
        int c = ci;
        while (c < nn && par[c] != j) ++c;
        if (irw[j] < 0 || c >= nn || st.r >= kTreeMaxRej) {
          act = 2;  // children exhausted (or a leaf): y ~ o_r with U(rid, j, SAMPLE)
          break;
        }
        ci = c + 1;
        const int32_t x = tok[c];
        double pv = s_cp[c], qv = s_cq[c];
        for (int s = 0; s < st.r; ++s) {  // o_r(x), q_r(x)
          const double dd = pv - qv;
          if (st.Zs[s] > 0.0) pv = (dd > 0.0 ? dd : 0.0) / st.Zs[s];
          qv = (x == st.xs[s]) ? 0.0 : qv * (double)st.qsc[s];
        }
        const double u = philox_u24(P.seed, rid, (uint32_t)c, P.step, kTagAccept);
        tm = fmin_(tm, (float)fabs(u - pv / qv));
        if (u * qv < pv) {  // accept: move to the child
          out[depth] = x;
          acc[depth] = c;
          depth++;
          j = c;
          need_init = true;
          continue;
        }
        // reject: o_{r+1} = norm(max(0, o_r - q_r)) needs its mass: a full pass
        st.xs[st.r] = x;
        st.qsc[st.r] = (qv < 1.0) ? (float)(1.0 / (1.0 - qv)) : 1.f;
        act = 1;
      }
#ifdef COSINE_TRACE
      {
        const unsigned long long t = tr_now();
        tr_acc[0] += t - tr_prev;  // slot 0 of the sums: the walk logic
        tr_prev = t;
        tr_act = act;
        tr_cnt[act]++;
      }
#endif
      s_act = act;
      s_node = j;
      s_err = err;
      s_Nd = (irw[j] >= 0) ? N : 0;
      if (act == 2) s_u = philox_u24(P.seed, rid, (uint32_t)j, P.step, kTagSample);
    }
    __syncthreads();
    const int act = s_act, jn = s_node, Nd = s_Nd;
    const TT* trow = (const TT*)P.target + ((int64_t)b * nn + jn) * P.ld_t;
    const TQ* drow = (const TQ*)P.draft + ((int64_t)b * P.I + (Nd ? irw[jn] : 0)) * N * P.ld_q;
    if (act == 4) {  // lazy: a visited node's data error (reading #23)
#ifdef COSINE_TRACE
      tr_flush();
#endif
      for (int c = tid; c < nn; c += kTreeBlock) { out[c] = -1; acc[c] = -1; }
      if (tid == 0) { P.accept_len[b] = -1; P.status[b] = s_err; }
      return;
    }
    if (act == 3) {  // lazy: node jn's row statistics (one pass) and its decisions (warp 0)
      tree_node_stats<TT, TQ, kLogits, NMAX>(T, b, jn, Nd, trow, drow, ring, s_full, s_empty, it, ntile,
                                             producer, s_rf, s_rd, s_rbad, s_ngx, s_ntok, s_nw, s_nsig,
                                             s_ndmax, &s_nzero, &s_nd, s_cp, s_cq, irw[jn]);
      if (tid == 0) s_have = jn;
      __syncthreads();
      continue;
    }
    // A pass: per-tile masses of the weights (mode, rr) into s_tile[0 .. ntile).  The producer
    // lane fills ring slots it .. it + ntile - 1; consumer warp w writes its partial of tile t to
    // s_parts[t][w]; the tile sums (fixed order) follow one block barrier.
    auto pass = [&](int mode, int rr) {
      if (producer) {
        if (lane == 0)
          for (int64_t t = 0; t < ntile; ++t) ring.fill(it + (uint32_t)t, t, P, trow, drow, Nd);
      } else {
        for (int64_t t = 0; t < ntile; ++t) {
          const uint32_t pos = it + (uint32_t)t;
          const int stg = (int)(pos % kTreeStages);
          mbar_wait_parity(&s_full[stg], (pos / kTreeStages) & 1u);
          const unsigned char* sb = ring.base + stg * Ring::kStageB;
          const int64_t g0 = t * kTG;
          const int tg = (int)min((int64_t)kTG, P.ngroups - g0);
          double m = 0.0;
          for (int g = tid; g < tg; g += kTreeThreads) {
            float w[8];
            tree_weights_s<TT, TQ, kLogits, NMAX>(st, mode, rr, sb, Nd, g, (int)((g0 + g) * kGroup), (int)P.V, w);
            m += (double)sum8(w);
          }
          m = warp_sum(m);
          if (lane == 0) {
            s_parts[t * kTreeWarps + warp] = m;
            mbar_arrive(&s_empty[stg]);  // this warp is done with the stage
          }
        }
      }
      it += (uint32_t)ntile;
      __syncthreads();
      for (int64_t t = tid; t < ntile; t += kTreeBlock) {
        double mt = 0.0;
        for (int w2 = 0; w2 < kTreeWarps; ++w2) mt += s_parts[t * kTreeWarps + w2];
        s_tile[t] = mt;
      }
    };
    if (act == 1) {  // Z_{r+1}: per-tile masses of max(0, o_r - q_r), kept for the final draw
      pass(0, st.r);
      __syncthreads();
      if (warp == 0) {
        const double Z = tile_total(s_tile, ntile, lane);
        if (lane == 0) {
        if (!(Z > 0.0)) deg = 1;  // all mass cancelled: o kept (reading #11)
        st.Zs[st.r] = Z;
        st.invZ[st.r] = (Z > 0.0) ? (float)(1.0 / Z) : 0.f;
        st.r++;
        }
      }
      __syncthreads();
      continue;
    }
    // act == 2: y ~ o_R of node jn (reading #10).  After R >= 1 rejections o_R is the residual of
    // the last pass, whose tile masses are still in s_tile: scan its crossing tile with weights
    // max(0, o_{R-1} - q_{R-1}) and t = u Z_R (the oracle's unnormalised form).  A leaf (the
    // bonus) or a degenerate last step needs a pass over o_R first.
    __shared__ int64_t s_tstar;
    __shared__ double s_tc, s_Z;
    __shared__ int s_mode, s_rr;
    __shared__ double s_ws[kTreeWarps];
    __shared__ int s_last[kTreeWarps];
    if (tid == 0) {
      const int R = st.r;
      const bool reuse = R >= 1 && st.Zs[R - 1] > 0.0;
      s_mode = reuse ? 0 : 1;
      s_rr = reuse ? R - 1 : R;
    }
    __syncthreads();
    const int mode = s_mode, rr = s_rr;
    if (mode == 1) {
      pass(1, rr);
      __syncthreads();
    }
    double Zf = 0.0;
    if (warp == 0) Zf = tile_total(s_tile, ntile, lane);
    if (tid == 0) {
      const double Z = Zf;
      const double t = s_u * Z;
      int64_t tstar = -1;
      double tc = 0.0, O = 0.0;
      for (int64_t t2 = 0; t2 < ntile && Z > 0.0; ++t2) {
        if (O + s_tile[t2] > t) { tstar = t2; tc = t - O; break; }
        O += s_tile[t2];
      }
      s_tstar = tstar;
      s_tc = tc;
      s_Z = Z;
      s_y = -1;
      s_margin = 0.f;
    }
    __syncthreads();
    if (s_tstar >= 0 && producer) {
      if (lane == 0) ring.fill(it, s_tstar, P, trow, drow, Nd);
      ++it;
    } else if (s_tstar >= 0) {  // the crossing tile: thread t holds kGPT consecutive groups; block scan
      constexpr int kGPT = (kTG + kTreeThreads - 1) / kTreeThreads;
      const int stg = (int)(it % kTreeStages);
      mbar_wait_parity(&s_full[stg], (it / kTreeStages) & 1u);
      ++it;
      const unsigned char* sb = ring.base + stg * Ring::kStageB;
      const int64_t g0 = s_tstar * kTG;
      const int tg = (int)min((int64_t)kTG, P.ngroups - g0);
      const double tc = s_tc;
      double s = 0.0;
      int last = -1;  // the last positive entry of this thread's groups (rounding fallback)
#pragma unroll
      for (int q = 0; q < kGPT; ++q) {
        const int gl = tid * kGPT + q;
        if (gl < tg) {
          float w[8];
          const int vb = (int)((g0 + gl) * kGroup);
          tree_weights_s<TT, TQ, kLogits, NMAX>(st, mode, rr, sb, Nd, gl, vb, (int)P.V, w);
          s += (double)sum8(w);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (w[e] > 0.f) last = vb + e;
        }
      }
      double incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double nb = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nb;
      }
      if (lane == 31) s_ws[warp] = incl;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
      if (lane == 0) s_last[warp] = last;
      consumer_sync();
      double base = 0.0;
      for (int w2 = 0; w2 < warp; ++w2) base += s_ws[w2];
      const double excl_w = __shfl_up_sync(0xffffffffu, incl, 1);
      const double lo = base + (lane == 0 ? 0.0 : excl_w), hi = base + incl;
      if (s > 0.0 && lo <= tc && tc < hi) {  // this thread's groups hold t: walk them in order
        double cum = lo;
        int y = -1, lastpos = -1;
        float mg = 0.f;
        for (int q = 0; q < kGPT && y < 0; ++q) {
          const int gl = tid * kGPT + q;
          if (gl >= tg) break;
          float w[8];
          const int vb = (int)((g0 + gl) * kGroup);
          tree_weights_s<TT, TQ, kLogits, NMAX>(st, mode, rr, sb, Nd, gl, vb, (int)P.V, w);
          for (int e = 0; e < 8; ++e) {
            const double prev = cum;
            cum += (double)w[e];
            if (w[e] > 0.f) lastpos = vb + e;
            if (cum > tc) { y = vb + e; mg = (float)(fmin(tc - prev, cum - tc) / s_Z); break; }
          }
        }
        if (y < 0) { y = lastpos; mg = 0.f; }
        s_y = y;
        s_margin = mg;
      }
      consumer_sync();
      if (tid == 0 && s_y < 0) {  // rounding fallback: the last positive entry of the tile (reading #10)
        int lst = -1;
        for (int w2 = 0; w2 < kTreeWarps; ++w2) lst = max(lst, s_last[w2]);
        s_y = lst;
        s_margin = 0.f;
      }
    }
    __syncthreads();
    if (tid == 0) {
      out[depth] = (int32_t)s_y;
      for (int c = depth + 1; c < nn; ++c) out[c] = -1;
      for (int c = depth; c < nn; ++c) acc[c] = -1;
      P.accept_len[b] = depth;
      tm = fmin_(tm, s_margin);
      P.status[b] = (deg ? COSINE_INFO_DEGENERATE_RESIDUAL : 0) | (tm < 1e-6f ? COSINE_INFO_NEAR_TIE : 0) |
                    (s_y < 0 ? 0xff : 0);
      if (P.dbg.tie_margin) P.dbg.tie_margin[b] = tm;
    }
#ifdef COSINE_TRACE
    tr_flush();
#endif
    return;
  }
}

}  // namespace cosine
