// cosine_split.cuh — the streaming verification kernels (Eq. 4 ARGMAX fusion).
//
// stats_kernel (A): one CTA per (unit, vocabulary chunk), unit = (request b, position
//   i <= gamma_b).  Each CTA streams its chunk of the unit's target logit row and N drafter
//   rows exactly once with 128-bit read-only loads, reduces them (online max / sum-exp of the
//   target, drafter row sums, greedy argmax) and writes a 128-byte partial record.
//   Register-lean (high occupancy = many loads in flight); never waits.
// decide_kernel (B1): one warp per unit — confidences and Eq. 4 fusion, acceptance
//   u * q(x*) < o(x*) — a programmatic dependent of A that waits per unit.
// resample_kernel (B2): the first rejection L and the final draw by inverse CDF over
//   norm(max(0, o - q)) of row L, or over o of the bonus row; waits per request.
// lazy_decide_kernel: the decisions of a lazy (NEXT-1) round.
#pragma once

#include "cosine_common.cuh"

namespace cosine {

template <bool B>
struct BoolTag {
  static constexpr bool value = B;
};


struct PartRec {  // one per (unit, chunk); 128 bytes
  float tmax;     // T > 0: chunk max logit; greedy: best value
  int32_t bad;    // bit0 target non-finite (greedy), bit1 negative drafter prob
  int64_t targ;   // greedy argmax (global index), -1 if none
  double tsum;    // sum 2^((l - tmax) k2) over the chunk
  float dmax[kMaxN];
  double dsum[kMaxN];
};

constexpr int kMaxPos = 65;  // draft positions per request (k <= 64) in kernel B
constexpr int kLazySpan = 2;  // positions per lazy round (NEXT-1)

enum SplitMode : int { kSplitVerify = 0, kSplitFuse = 1, kSplitSample = 2 };

// Phase timestamps for latency studies (tools/tiny_trace.py builds the library with
// -DCOSINE_TRACE; in the product build the macro is empty).
#ifdef COSINE_TRACE
#define COSINE_TRACE_AT(P, slot)                                                      \
  do {                                                                                \
    if ((P).trace && threadIdx.x == 0) {                                              \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      (P).trace[(size_t)blockIdx.x * 16 + (slot)] = t_;                                \
    }                                                                                 \
  } while (0)
#else
#define COSINE_TRACE_AT(P, slot) ((void)0)
#endif

struct SplitParams {
  int mode;  // kSplitVerify (cosine_verify_batch / _lazy / _tree), kSplitFuse, kSplitSample
  // cosine_fuse_drafts outputs
  int32_t* fuse_tokens;
  float* fuse_w;
  float* fuse_sig;
  float* fused_q;
  int64_t ld_fq;
  // cosine_sample_residual inputs / outputs (mode kSplitSample: request b = one row group)
  const float* row_max;
  const float* row_sumexp;
  const float* w_in;
  const float* norm_in;
  const uint32_t* node_ids;
  int32_t* out_token;
  int B, k, N;
  int64_t V, ld_t, ld_q, ngroups, gfull;
  int C;          // CTAs per unit (kernel A)
  int64_t cg;     // groups per chunk (kernel A)
  int C2;         // cluster size (kernel B)
  int64_t cg2;    // groups per chunk (kernel B)
  float k2f;
  double k2d;
  int greedy, weight_mode, select;
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
  PartRec* parts;
  struct PosDec* pdec;
  int32_t* counters;  // [B] CTAs of a request done (kernel B), reset by the last one
  // fine-grained dependencies (single-GPU linear path): kernels B1 and B2 are programmatic
  // dependents scheduled into the previous kernel's tail wave; B1 waits for its unit's C chunk
  // records, B2 for its request's g + 1 decisions, instead of for the whole previous grid
  int fused;
  int ucount;         // stats_kernel counts each chunk on ucnt (fused split path; sharded records)
  int32_t* ucnt;      // [B][k+1] chunk CTAs of a unit done (kernel A), reset by kernel B1
  int32_t* dcnt;      // [B] units of a request decided (kernel B1), reset by the request's last B2 CTA
  // lazy verification (NEXT-1, cosine_verify_batch_lazy): lazy = r + 1 in round r, which
  // streams position r of the requests still verifying (0 = off); lz[b] = 0 while request b
  // verifies, -1 once it stopped
  int lazy;
  int lazy_span;  // positions per lazy round
  int32_t* lz;
  double* segsum;  // [B][nseg] residual / bonus mass per 256-group segment
  int64_t nseg;
  // SAMPLE selection over probability drafts: the statistics pass also writes the drafter row
  // sums of every kSliceGroups-group slice of its chunk, slices[((unit * C + chunk) * nsl + s) * N + n]
  // (fp32 warp sums), so that the draw x* ~ q locates its slice without re-reading the chunk
  float* slices;
  int64_t nsl;     // slices per chunk (ceil(cg / kSliceGroups))
  unsigned long long* trace;  // instrumentation builds only (-DCOSINE_TRACE): [grid][16] timestamps
  int spr;         // B2a CTAs per request
  int tpc;         // tiles per B2 CTA (<= kSegTilesPerCta)
  int b_off, nb;   // this launch covers requests [b_off, b_off + nb) (batch pipelining)
  // tree mode (cosine_verify_tree): a unit is a node (b, j); rows via internal_row
  int tree, nn, I;           // nodes per request (J + 1), internal (drafter) rows per request
  const int32_t* irow;       // [B][nn] drafter row of node j, -1 for a leaf
  // vocabulary-sharded mode (nranks > 1, cosine_shard.cuh): this rank holds columns
  // [v0, v0 + V) of every row of a Vg-wide vocabulary; V, ngroups, gfull are the local ones
  int shard, G, rank;
  int64_t v0, Vg;
  int rec_words;             // 32-bit words per ShardRec (depends on N)
  uint32_t* rec_send;        // [units][rec_words] this rank's records
  const uint32_t* rec_all;   // [G][units][rec_words] every rank's (all-gather)
  double* zsend;             // [B] local mass of the final draw
  const double* zall;        // [G][B]
  struct YRec* ysend;        // [B] the owner's token (-1 elsewhere)
  const struct YRec* yall;   // [G][B]
  // in-kernel exchange over NVLink peer memory (p2p = 1, replaces the three NCCL all-gathers):
  // the kernel that produces a record / mass / token writes it straight into every rank's
  // gather buffer (peer pointers of this call, rank-major layout as the all-gather's) and counts
  // it on every rank's arrival counter [3] (rec, z, y); the consumer waits until its own counter
  // reaches the call's cumulative target tgt[x]
  int p2p;
  uint32_t* rec_peer[8];
  double* z_peer[8];
  struct YRec* y_peer[8];
  unsigned long long* cnt_peer[8];
  unsigned long long* cnt_own;
  unsigned long long tgt[3];
};


// One warp scans groups [gb, ge) in vocabulary order: smallest v with C(v) > tc, C the running
// sum of w from gb; rounding fallback = last v with w(v) > 0 (reading #10).  All lanes return y.
template <typename TT, typename TQ, bool kLogits, int NMAX, typename PP>
__device__ __forceinline__ int64_t warp_scan_range(const PP& P, const Decision& d, int kind,
                                                   const TT* trow, const TQ* drow, int Nd, int64_t gb,
                                                   int64_t ge, double tc, double Z, float* margin) {
  const int lane = threadIdx.x & 31;
  double base = 0.0;
  for (int64_t t0 = gb; t0 < ge; t0 += 32) {
    const int64_t gi = t0 + lane;
    float w[8];
    double s = 0.0;
    if (gi < ge) {
      group_weights<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, gi, w);
      s = (double)sum8(w);
    }
    double incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double nb = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += nb;
    }
    const double excl = base + incl - s;
    const bool hit = gi < ge && s > 0.0 && excl <= tc && tc < excl + s;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (m) {
      const int src = __ffs(m) - 1;
      int64_t y = -1;
      float mg = 0.f;
      if (lane == src) {
        double cum = excl;
        int ef = -1;
        for (int e = 0; e < 8; ++e) {
          const double prev = cum;
          cum += (double)w[e];
          if (cum > tc) {
            ef = e;
            mg = (float)(fmin(tc - prev, cum - tc) / Z);
            break;
          }
        }
        if (ef < 0)
          for (int e = 7; e >= 0; --e)
            if (w[e] > 0.f) { ef = e; break; }
        y = gi * kGroup + ef;
      }
      y = __shfl_sync(0xffffffffu, y, src);
      *margin = __shfl_sync(0xffffffffu, mg, src);
      return y;
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
  int64_t last = -1;
  for (int64_t gi = gb + lane; gi < ge; gi += 32) {
    float w[8];
    group_weights<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, gi, w);
    for (int e = 0; e < 8; ++e)
      if (w[e] > 0.f) last = max(last, gi * kGroup + e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
  *margin = 0.f;
  return last;
}

// ============================== kernel A ==============================
constexpr int kSliceGroups = 32;  // groups per slice of the SAMPLE slice sums (stats_kernel<..., kSlices>)

// K per-lane values -> their K warp sums in K - 1 + 5 - log2(K) shuffles instead of 5 K (a
// transposed reduction: each level halves the values a lane holds); lane l returns the sum of
// value l / (32 / K).
template <int K>
__device__ __forceinline__ float warp_sums_scatter(const float (&v)[K]) {
  static_assert(K >= 1 && K <= 32 && (K & (K - 1)) == 0, "K: a power of two <= 32");
  const int lane = threadIdx.x & 31;
  float cur[K];
#pragma unroll
  for (int j = 0; j < K; ++j) cur[j] = v[j];
  int o = 16;
#pragma unroll
  for (int w = K; w > 1; w >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < w / 2; ++j) {
      const float send = up ? cur[j] : cur[j + w / 2];
      const float keep = up ? cur[j + w / 2] : cur[j];
      cur[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (; o > 0; o >>= 1) cur[0] += __shfl_xor_sync(0xffffffffu, cur[0], o);
  return cur[0];
}

// Resident CTAs per SM of the streaming kernels: register-lean (40 registers) for bf16 with
// N <= 4, so that 48 warps of 128-bit loads are in flight per SM.
template <typename TT, typename TQ, int NMAX, bool kLogits = false>
constexpr int stats_occupancy() {
  // logit drafter rows keep a running max per drafter and are ex2-bound: 48 registers, 5 CTAs
  return (NMAX <= 4 && sizeof(TT) == 2 && sizeof(TQ) == 2) ? (kLogits ? 5 : 6) : 4;
}

// One CTA's share of a unit: chunk `rank` of the unit's target row and N drafter rows, streamed
// once; writes the chunk's partial record.  Returns the unit's record index, or -1 when the CTA
// has no rows (position past gamma_b, bad gamma_b, or a stopped lazy request).  Ends with the
// record written by warp 0 (no trailing barrier).
template <typename TT, typename TQ, bool kLogits, int NMAX, bool kSlices = false, bool kRowU4 = true>
__device__ __forceinline__ int64_t stats_body(const SplitParams& P, int64_t unit, int rank) {
  static_assert(!(kSlices && kLogits), "slice sums are kept for probability drafts only");
  const int C = P.C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = P.N;
  int Nd;
  const TT* trow;
  const TQ* drow;
  int64_t gu;  // the unit's index in the partial-record array
  if (P.mode == kSplitFuse) {  // cosine_fuse_drafts: unit (b, i < k), drafter rows only
    // (no target row: the "target" statistics of the record are taken over drafter row 0 —
    // its second load of each group is an L2 hit — and ignored by fuse_decide_kernel; this
    // keeps the streaming loop free of a target-present branch)
    const int b = (int)(unit / P.k), i = (int)(unit % P.k);
    Nd = N;
    drow = (const TQ*)P.draft + ((int64_t)b * P.k + i) * N * P.ld_q;
    trow = reinterpret_cast<const TT*>(drow);
    gu = unit;
  } else if (P.mode == kSplitSample) {  // cosine_sample_residual: unit b = one target row (+ N drafter rows)
    Nd = P.draft ? N : 0;
    trow = (const TT*)P.target + unit * P.ld_t;
    drow = (const TQ*)P.draft + unit * N * P.ld_q;
    gu = unit;
  } else if (P.tree) {  // node (b, j): target row j, the N drafter rows of its internal row (if any)
    const int b = (int)(unit / P.nn);
    const int ir = P.irow[unit];
    Nd = (ir >= 0 && ir < P.I) ? N : 0;
    trow = (const TT*)P.target + unit * P.ld_t;
    drow = (const TQ*)P.draft + ((int64_t)b * P.I + (Nd ? ir : 0)) * N * P.ld_q;
    gu = unit;
  } else {
    int b, i;
    if (P.lazy) {  // lazy round (NEXT-1): positions r0 .. r0+span-1 of the requests still verifying
      b = (int)(unit / P.lazy_span);
      i = P.lazy - 1 + (int)(unit % P.lazy_span);
      if (P.lazy > 1 && P.lz[b] != 0) return -1;
    } else {
      b = P.b_off + (int)(unit / (P.k + 1));
      i = (int)(unit % (P.k + 1));
    }
    const int g = P.draft_len ? P.draft_len[b] : P.k;
    if (g < 1 || g > P.k || i > g) return -1;  // rows past gamma_b are never read
    Nd = (i < g) ? N : 0;
    gu = (int64_t)b * (P.k + 1) + i;
    trow = (const TT*)P.target + gu * P.ld_t;
    drow = (const TQ*)P.draft + ((int64_t)b * P.k + i) * N * P.ld_q;
  }

  __shared__ float s_wf[kWarps][1 + kMaxN];
  __shared__ float s_wv[kWarps];
  __shared__ int64_t s_wi[kWarps];
  __shared__ double s_wd[kWarps][1 + kMaxN];
  __shared__ int32_t s_wbad[kWarps];

  const bool greedy = !kSlices && P.greedy != 0;  // (the slice variant runs at T > 0 only)
  const float k2 = P.k2f;
  float tmx = kNegBig, tmk = kNegBig, ts = 0.f;  // running max, fl(max * k2), sum 2^(l k2 - tmk)
  float tb = -INFINITY;
  int64_t ti = -1;
  bool tbad = false, dneg = false;
  float dm[NMAX], dmk[NMAX], ds[NMAX];
#pragma unroll
  for (int n = 0; n < NMAX; ++n) { dm[n] = kNegBig; dmk[n] = kNegBig; ds[n] = 0.f; }
  float dacc = 0.f;  // kSlices: this lane's drafter's running slice total (see below)
  const int64_t gb = (int64_t)rank * P.cg;
  const int64_t ge = min(P.ngroups, gb + P.cg);
  const int64_t gfe = min(ge, P.gfull);  // full groups of the chunk

  auto t_step = [&](const float (&f)[8], int64_t gi) {
    if (greedy) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (f[e] > tb) { tb = f[e]; ti = gi * kGroup + e; }
        tbad |= !(f[e] <= 3.402823466e+38f);
      }
    } else {
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
    }
  };
  auto d_step = [&](int n, const float (&f)[8]) {
    if (kLogits) {
      const float gm = max8(f);
      if (gm > dm[n]) {
        const float nmk = gm * k2;
        ds[n] *= ex2(dmk[n] - nmk);
        dm[n] = gm;
        dmk[n] = nmk;
      }
      float e8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) e8[e] = ex2(fmaf(f[e], k2, -dmk[n]));
      ds[n] += sum8(e8);
    } else {
      ds[n] += sum8(f);
    }
  };

  if (kRowU4 && Nd == 0) {
    // a target row alone (the bonus position, a tree leaf): four groups per thread in flight,
    // as many bytes as the (1 + N)-row units keep in flight (one group per row) — with one load
    // per step such a CTA held its slot ~75% as long for ~20% of the bytes.  Same per-thread
    // order of the groups as the loop below.
    int64_t gi = gb + tid;
    for (; gi + 3 * kThreads < gfe; gi += 4 * kThreads) {
      Group<TT> t4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t4[u].load(trow, gi + u * kThreads);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float f[8];
        t4[u].unpack(f);
        t_step(f, gi + u * kThreads);
      }
    }
    for (; gi < gfe; gi += kThreads) {
      Group<TT> tv;
      tv.load(trow, gi);
      float f[8];
      tv.unpack(f);
      t_step(f, gi);
    }
  } else if constexpr (kSlices) {
    // the same stream in warp-contiguous slices: warp w covers slices s = w, w + 8, ... of
    // kSliceGroups consecutive groups (two coalesced 32-group steps each), whose drafter sums it
    // writes (a transposed warp reduction: one shuffle tree for all N sums)
    float* sl = P.slices + (gu * C + rank) * P.nsl * N;
    // (the chunk's drafter sums are the sums of its slices: lane l accumulates the slice totals
    // of drafter l / (32 / NMAX), so no per-thread drafter sums stay live across the loop)
    for (int64_t s0 = gb + (int64_t)kSliceGroups * warp; s0 < gfe; s0 += (int64_t)kSliceGroups * kWarps) {
      float sn[NMAX];
#pragma unroll
      for (int n = 0; n < NMAX; ++n) sn[n] = 0.f;
#pragma unroll
      for (int h = 0; h < kSliceGroups; h += 32) {
        const int64_t gi = s0 + h + lane;
        if (gi < gfe) {
          Group<TT> tv;
          Group<TQ> dv[NMAX];
          tv.load(trow, gi);
#pragma unroll
          for (int n = 0; n < NMAX; ++n)
            if (n < Nd) dv[n].load(drow + (int64_t)n * P.ld_q, gi);
          float f[8];
          tv.unpack(f);
          t_step(f, gi);
#pragma unroll
          for (int n = 0; n < NMAX; ++n) {
            if (n < Nd) {
              dv[n].unpack(f);
              if (dv[n].any_sign()) {
#pragma unroll
                for (int e = 0; e < 8; ++e) dneg |= (f[e] < 0.f);
              }
              sn[n] += sum8(f);
            }
          }
        }
      }
      const float tot = warp_sums_scatter<NMAX>(sn);
      dacc += tot;
      const int idx = lane / (32 / NMAX);
      if (lane % (32 / NMAX) == 0 && idx < Nd) sl[((s0 - gb) / kSliceGroups) * N + idx] = tot;
    }
  } else {
    for (int64_t gi = gb + tid; gi < gfe; gi += kThreads) {
      Group<TT> tv;
      Group<TQ> dv[NMAX];
      tv.load(trow, gi);
#pragma unroll
      for (int n = 0; n < NMAX; ++n)
        if (n < Nd) dv[n].load(drow + (int64_t)n * P.ld_q, gi);
      float f[8];
      tv.unpack(f);
      t_step(f, gi);
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n < Nd) {
          dv[n].unpack(f);
          if (!kLogits && dv[n].any_sign()) {
#pragma unroll
            for (int e = 0; e < 8; ++e) dneg |= (f[e] < 0.f);
          }
          d_step(n, f);
        }
      }
    }
  }
  if (gfe < ge && tid == (int)((gfe - gb) % kThreads)) {  // the row's partial last group
    const int64_t gi = gfe;
    float f[8];
    load_partial(trow, gi, P.V, -INFINITY, f);
    t_step(f, gi);
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      if (n < Nd) {
        load_partial(drow + (int64_t)n * P.ld_q, gi, P.V, kLogits ? -INFINITY : 0.f, f);
        if (!kLogits) {
#pragma unroll
          for (int e = 0; e < 8; ++e) dneg |= (f[e] < 0.f);
        }
        d_step(n, f);
      }
    }
  }

  // ---------------- CTA reduction -> partial record ----------------
  float tmw = kNegBig, tbw = tb;
  int64_t tiw = ti;
  if (greedy) warp_argmax(tbw, tiw);
  else tmw = warp_max(tmx);
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
#pragma unroll
  for (int w = 0; w < kWarps; ++w) Mc = fmaxf(Mc, s_wf[w][0]);
  // thread sums are relative to 2^(fl(m k2)); rescale exactly (fp64) to 2^(Mc k2)
  double tsd = 0.0;
  if (!greedy && ts != 0.f) tsd = (double)ts * exp2((double)tmk - (double)Mc * (double)k2);
  tsd = warp_sum(tsd);
  double dsd[NMAX];
#pragma unroll
  for (int n = 0; n < NMAX; ++n) {
    dsd[n] = 0.0;
    if (n < Nd) {
      if (kLogits) {
        float dMc = kNegBig;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) dMc = fmaxf(dMc, s_wf[w][1 + n]);
        if (ds[n] != 0.f) dsd[n] = (double)ds[n] * exp2((double)dmk[n] - (double)dMc * (double)k2);
        dsd[n] = warp_sum(dsd[n]);
      } else if (kSlices) {  // the warp's slice totals (+ the partial group's thread sum)
        dsd[n] = (double)__shfl_sync(0xffffffffu, dacc, n * (32 / NMAX)) + warp_sum((double)ds[n]);
      } else {
        dsd[n] = warp_sum((double)ds[n]);
      }
    }
  }
  const int bad = (__any_sync(0xffffffffu, tbad) ? 1 : 0) | (__any_sync(0xffffffffu, dneg) ? 2 : 0);
  if (lane == 0) {
    s_wd[warp][0] = tsd;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) s_wd[warp][1 + n] = dsd[n];
    s_wbad[warp] = bad;
  }
  __syncthreads();
  if (tid < 32) {  // warp 0 assembles the record: lane j owns field j
    PartRec* rec = P.parts + gu * C + rank;
    if (lane == 0) {
      float bv = Mc;
      int64_t bi = -1;
      if (greedy) {
        bv = -INFINITY;
        for (int w = 0; w < kWarps; ++w) {
          const float v = s_wv[w];
          const int64_t ix = s_wi[w];
          if (ix >= 0 && (bi < 0 || v > bv || (v == bv && ix < bi))) { bv = v; bi = ix; }
        }
      }
      double t = 0.0;
      int bd = 0;
      for (int w = 0; w < kWarps; ++w) { t += s_wd[w][0]; bd |= s_wbad[w]; }
      rec->tmax = bv;
      rec->targ = bi;
      rec->tsum = t;
      rec->bad = bd;
    } else if (lane <= kMaxN) {
      const int n = lane - 1;
      float mx = kNegBig;
      double sacc = 0.0;
      if (n < NMAX) {
        for (int w = 0; w < kWarps; ++w) { mx = fmaxf(mx, s_wf[w][1 + n]); sacc += s_wd[w][1 + n]; }
      }
      rec->dmax[n] = mx;
      rec->dsum[n] = sacc;
    }
  }
  return gu;
}

template <typename TT, typename TQ, bool kLogits, int NMAX, bool kSlices = false>
__global__ void __launch_bounds__(kThreads, (stats_occupancy<TT, TQ, NMAX, kLogits>()))
    stats_kernel(const SplitParams P) {
  // every CTA of this grid is resident or done once all passed this point: kernel B (launched
  // as a programmatic dependent) may then be scheduled into the tail wave (it waits per unit)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  COSINE_TRACE_AT(P, 0);
  const int64_t gu =
      stats_body<TT, TQ, kLogits, NMAX, kSlices>(P, blockIdx.x / P.C, (int)(blockIdx.x % P.C));
  if ((P.fused || P.ucount) && gu >= 0) {  // count this chunk for the unit (the next kernel waits per unit)
    __syncthreads();
    COSINE_TRACE_AT(P, 1);
    if (threadIdx.x == 0) red_release_add(&P.ucnt[gu], 1);  // the record before the count
  }
}

// ============================== kernel B ==============================
struct PosDec {  // decisions of one position (shared memory of every CTA of the cluster)
  int32_t status, accept, xstar;
  int64_t amax;
  float m_fa, M;
  double S, px, qx, u;
  float a[kMaxN], dm[kMaxN];
  float sig[kMaxN], c[kMaxN], w[kMaxN];
};

__device__ __forceinline__ void init_posdec(PosDec& pd) {
  pd.status = 0; pd.accept = 1; pd.xstar = -1; pd.amax = -1; pd.m_fa = INFINITY; pd.M = 0.f; pd.S = 0.0;
  pd.px = pd.qx = pd.u = NAN;
  for (int n = 0; n < kMaxN; ++n) { pd.a[n] = 0.f; pd.dm[n] = 0.f; pd.sig[n] = NAN; pd.c[n] = NAN; pd.w[n] = NAN; }
}

__device__ __forceinline__ void write_pos_debug(const SplitParams& P, int b, int i, bool has_d, const PosDec& pd) {
  const cosine_debug_t& D = P.dbg;
  const int64_t unit = (int64_t)b * (P.k + 1) + i;
  if (D.row_max) D.row_max[unit] = pd.M;
  if (D.row_sumexp) D.row_sumexp[unit] = P.greedy ? 0.f : (float)pd.S;
  if (has_d) {
    const int64_t o1 = (int64_t)b * P.k + i;
    if (D.p_x) D.p_x[o1] = (float)pd.px;
    if (D.q_x) D.q_x[o1] = (float)pd.qx;
    if (D.accept_u) D.accept_u[o1] = (float)pd.u;
    if (D.fused_tokens) D.fused_tokens[o1] = pd.xstar;
    for (int n = 0; n < P.N; ++n) {
      if (D.draft_norm) D.draft_norm[o1 * P.N + n] = pd.sig[n];
      if (D.conf) D.conf[o1 * P.N + n] = pd.c[n];
      if (D.weights) D.weights[o1 * P.N + n] = pd.w[n];
    }
  }
}

// A unit's combined row statistics, in every lane of a decision warp; drafter n's values in
// lane n (no per-drafter arrays: a lane-0 sequential decision with local arrays costs ~7 us of
// latency per position, which dominates small batches and the decision kernels' tails).
struct UnitStats {
  float M;       // T > 0: row max; greedy: the best value
  double S;      // sum 2^((l - M) k2) (0 when greedy)
  int64_t amax;  // greedy argmax, -1 otherwise
  bool t_nf, t_empty, d_nf, d_empty, tok_bad;
  double sig;    // lane n < N: sigma_n (PROBS: the row sum; LOGITS: sum-exp at its max)
  float dmx;     // lane n < N: LOGITS row max (kNegBig for PROBS)
};

// One warp: the gathers of the drafters' own tokens into s_gxw / s_tokw (lane m * N + n:
// d_m(X_n), m == N: l(X_n); `diag_only`: d_n(X_n) only) and the combination of the unit's C
// chunk records (chunk r in lane r, fixed-order shuffle reductions, fp64).  `has_t` = false:
// cosine_fuse_drafts units (b * k + i, no target row).
template <typename TT, typename TQ, bool kLogits>
__device__ __forceinline__ UnitStats warp_combine(const SplitParams& P, int b, int i, bool has_d, bool diag_only,
                                                  float* s_gxw, int32_t* s_tokw, bool has_t = true) {
  const int lane = threadIdx.x & 31;
  const int N = P.N, C = P.C;
  const int64_t unit = has_t ? (int64_t)b * (P.k + 1) + i : (int64_t)b * P.k + i;
  const bool greedy = P.greedy != 0;
  const double k2 = (double)P.k2f;
  const int ng = has_d ? N * (N + 1) : 0;
  if (lane < ng) {
    const int n = lane % N, m = lane / N;
    const int32_t tk = P.draft_tokens[((int64_t)b * P.k + i) * N + n];
    float v = 0.f;
    if (tk >= 0 && (int64_t)tk < P.V && (!diag_only || m == n) && (m < N || has_t)) {
      if (m < N) v = load_one((const TQ*)P.draft + (((int64_t)b * P.k + i) * N + m) * P.ld_q, tk);
      else v = load_one((const TT*)P.target + ((int64_t)b * (P.k + 1) + i) * P.ld_t, tk);
    }
    s_gxw[m * kMaxN + n] = v;
    if (m == 0) s_tokw[n] = tk;
  }
  COSINE_TRACE_AT(P, 8);
  const PartRec* parts = P.parts + unit * C;  // L2 reads (written by other CTAs)
  const bool own = lane < C;
  const float tmax = own ? __ldcg(&parts[lane].tmax) : kNegBig;
  const int bad = __reduce_or_sync(0xffffffffu, own ? __ldcg(&parts[lane].bad) : 0);
  UnitStats st;
  st.M = 0.f;
  st.S = 0.0;
  st.amax = -1;
  st.t_nf = st.t_empty = st.d_nf = st.d_empty = st.tok_bad = false;
  st.sig = NAN;
  st.dmx = kNegBig;
  if (!has_t) {
    // no target row (its record fields are ignored)
  } else if (greedy) {
    float bv = own ? tmax : -INFINITY;
    int64_t bi = own ? (int64_t)__ldcg((const long long*)&parts[lane].targ) : -1;
    warp_argmax(bv, bi);
    st.t_nf = (bad & 1) != 0;
    st.t_empty = (bi < 0);
    st.amax = bi;
    st.M = bv;
  } else {
    st.M = warp_max(tmax);
    const double tsum = own ? __ldcg(&parts[lane].tsum) : 0.0;
    st.S = warp_sum(tsum != 0.0 ? tsum * exp2((double)tmax * k2 - (double)st.M * k2) : 0.0);
    st.t_nf = !isfinite(st.S) || !isfinite(st.M);
    st.t_empty = !st.t_nf && !(st.S > 0.0);
  }
  if (has_d) {
    st.d_nf = (bad & 2) != 0;
    for (int n = 0; n < N; ++n) {
      double sv;
      float mx = kNegBig;
      const double ds = own ? __ldcg(&parts[lane].dsum[n]) : 0.0;
      if (kLogits) {
        const float dmr = own ? __ldcg(&parts[lane].dmax[n]) : kNegBig;
        mx = warp_max(dmr);
        sv = warp_sum(ds != 0.0 ? ds * exp2((double)dmr * k2 - (double)mx * k2) : 0.0);
        if (!isfinite(mx)) st.d_nf = true;
      } else {
        sv = warp_sum(ds);
      }
      if (lane == n) { st.sig = sv; st.dmx = mx; }
      if (!isfinite(sv)) st.d_nf = true;
      else if (!(sv > 0.0)) st.d_empty = true;
    }
  }
  __syncwarp();
  if (has_d) {
    const int32_t t = lane < N ? s_tokw[lane] : 0;
    st.tok_bad = __any_sync(0xffffffffu, lane < N && (t < 0 || (int64_t)t >= P.V));
  }
  COSINE_TRACE_AT(P, 9);
  return st;
}

// One warp decides position i of request b from its combined statistics (Eq. 4 fusion
// P:406-411, acceptance P:130-131), lane-parallel: lane n holds drafter n's sigma_n and
// confidence c_n, the fusion argmax / second best / weight sum are shuffle reductions, lane n
// writes drafter n's fields of *out (lane 0 the scalars) and of the diagnostics.
// `w_sample` (SAMPLE selection, cosine_fuse_drafts): stop after the weights — x* is the
// caller's draw — and leave w_n in w_sample[n] (and sigma_n, the LOGITS row max in sig_out /
// dmax_out).  s_gxw / s_tokw / st as warp_combine leaves them (or the sharded records).  Ends
// with __syncwarp().
template <bool kLogits>
__device__ __forceinline__ void warp_decide_core(const SplitParams& P, int b, int i, bool has_d, const UnitStats& st,
                                                 const float* s_gxw, const int32_t* s_tokw, PosDec* out,
                                                 bool write_debug, double* w_sample = nullptr,
                                                 double* sig_out = nullptr, float* dmax_out = nullptr) {
  const int lane = threadIdx.x & 31;
  const int N = P.N;
  const int64_t unit = (int64_t)b * (P.k + 1) + i;
  const bool greedy = P.greedy != 0;
  const double k2 = (double)P.k2f;
  const bool dl = lane < N;  // this lane holds a drafter
  const double sig_l = st.sig;
  const float dmx_l = st.dmx;
  if (dl && sig_out) sig_out[lane] = sig_l;
  if (dl && dmax_out) dmax_out[lane] = dmx_l;
  int stc = st.tok_bad ? COSINE_REQ_TOKEN_OUT_OF_RANGE
                       : ((st.t_nf || st.d_nf) ? COSINE_REQ_NONFINITE_INPUT
                                                : ((st.t_empty || st.d_empty) ? COSINE_REQ_EMPTY_ROW : 0));
  // q_n(x) of a gathered drafter value (PROBS: d / sigma; LOGITS: softmax at the same k2), lane n
  auto qval = [&](double dv) {
    return kLogits ? exp2(dv * k2 - (double)dmx_l * k2) / sig_l : dv / sig_l;
  };
  double c_l = 0.0;  // c_{n,i} = q_{n,i}(X_{n,i})
  if (!stc && has_d) {
    if (dl) c_l = qval((double)s_gxw[lane * kMaxN + lane]);
    if (__any_sync(0xffffffffu, dl && c_l == 0.0)) stc = COSINE_REQ_ZERO_PROB_DRAFT;
  }
  const bool filled = !stc && has_d;
  COSINE_TRACE_AT(P, 10);
  int accept = 1, xstar = -1;
  float m_fa = INFINITY;
  double px = NAN, qx = NAN, u = NAN, w_l = NAN;
  if (filled) {
    // Eq. 4: n* = argmax_n c_n, ties -> lowest n; fused weights (reading #2)
    double bc = dl ? c_l : -1.0;
    int bn = dl ? lane : 1 << 30;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const int on = __shfl_xor_sync(0xffffffffu, bn, o);
      if (oc > bc || (oc == bc && on < bn)) { bc = oc; bn = on; }
    }
    const int ns = bn;
    double second = (dl && lane != ns) ? c_l : -1.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) second = fmax(second, __shfl_xor_sync(0xffffffffu, second, o));
    m_fa = (N > 1) ? (float)((bc - second) / bc) : INFINITY;
    if (P.weight_mode == COSINE_W_CONF) {
      const double sc = warp_sum(dl ? c_l : 0.0);
      w_l = dl ? c_l / sc : 0.0;
    } else if (P.weight_mode == COSINE_W_UNIFORM) {
      w_l = dl ? 1.0 / (double)N : 0.0;
    } else {
      w_l = (lane == ns) ? 1.0 : 0.0;
    }
    xstar = s_tokw[ns];
    if (w_sample) {  // x* is the caller's (SAMPLE: a draw from q; cosine_fuse_drafts)
      // n* matters for the ARGMAX token and for WINNER weights only
      if (P.weight_mode != COSINE_W_WINNER && P.select != COSINE_SEL_ARGMAX) m_fa = INFINITY;
      if (dl) w_sample[lane] = w_l;
    } else {
      if (P.weight_mode == COSINE_W_POINT) {
        qx = 1.0;
      } else {
        qx = warp_sum(dl ? w_l * qval((double)s_gxw[lane * kMaxN + ns]) : 0.0);
      }
      COSINE_TRACE_AT(P, 11);
      u = philox_u24(P.seed, P.rids[b], (uint32_t)(i + 1), P.step, kTagAccept);
      COSINE_TRACE_AT(P, 12);
      if (greedy) {
        accept = ((int64_t)xstar == st.amax);
      } else {
        // acceptance u * q(x*) < o(x*), i.e. u < min(1, o/q)
        px = exp2((double)s_gxw[N * kMaxN + ns] * k2 - (double)st.M * k2) / st.S;
        accept = (u * qx < px);
        m_fa = fmin_(m_fa, (float)fabs(u - px / qx));
      }
    }
  }
  COSINE_TRACE_AT(P, 13);
  // ---- the decision record: lane n < kMaxN writes drafter n's fields, lane 0 the scalars ----
  if (lane < kMaxN) {
    const bool mine = filled && dl;
    out->a[lane] = mine ? (float)(w_l / sig_l) : 0.f;
    out->dm[lane] = mine ? dmx_l : 0.f;
    out->sig[lane] = mine ? (float)sig_l : NAN;
    out->c[lane] = mine ? (float)c_l : NAN;
    out->w[lane] = mine ? (float)w_l : NAN;
  }
  if (lane == 0) {
    out->status = stc;
    out->accept = accept;
    out->xstar = xstar;
    out->amax = st.amax;
    out->m_fa = m_fa;
    out->M = st.M;
    out->S = st.S;
    out->px = px;
    out->qx = qx;
    out->u = u;
  }
  if (write_debug) {
    const cosine_debug_t& D = P.dbg;
    const int64_t o1 = (int64_t)b * P.k + i;
    if (lane == 0) {
      if (D.row_max) D.row_max[unit] = st.M;
      if (D.row_sumexp) D.row_sumexp[unit] = greedy ? 0.f : (float)st.S;
      if (has_d) {
        if (D.p_x) D.p_x[o1] = (float)px;
        if (D.q_x) D.q_x[o1] = (float)qx;
        if (D.accept_u) D.accept_u[o1] = (float)u;
        if (D.fused_tokens) D.fused_tokens[o1] = xstar;
      }
    }
    if (has_d && dl) {
      if (D.draft_norm) D.draft_norm[o1 * N + lane] = filled ? (float)sig_l : NAN;
      if (D.conf) D.conf[o1 * N + lane] = filled ? (float)c_l : NAN;
      if (D.weights) D.weights[o1 * N + lane] = filled ? (float)w_l : NAN;
    }
  }
  __syncwarp();
  COSINE_TRACE_AT(P, 14);
}

// One warp decides position i of request b (split path): warp_combine + warp_decide_core.
template <typename TT, typename TQ, bool kLogits>
__device__ __forceinline__ void warp_decide(const SplitParams& P, int b, int i, int g, float* s_gxw,
                                            int32_t* s_tokw, PosDec* out, bool write_debug) {
  const bool has_d = i < g;
  const UnitStats st = warp_combine<TT, TQ, kLogits>(P, b, i, has_d, false, s_gxw, s_tokw);
  warp_decide_core<kLogits>(P, b, i, has_d, st, s_gxw, s_tokw, out, write_debug);
}

// Kernel B1 (split path): one warp per (request, position) -> PosDec in global memory (+
// diagnostics); a programmatic dependent of stats_kernel that waits per unit (device counter).
template <typename TT, typename TQ, bool kLogits>
__global__ void __launch_bounds__(kThreads) decide_kernel(const SplitParams P) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t unit = (int64_t)blockIdx.x * kWarps + warp;
  __shared__ float s_gx[kWarps][(kMaxN + 1) * kMaxN];
  __shared__ int32_t s_tok[kWarps][kMaxN];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (unit >= (int64_t)P.B * (P.k + 1)) return;
  const int b = (int)(unit / (P.k + 1)), i = (int)(unit % (P.k + 1));
  const int g = P.draft_len ? P.draft_len[b] : P.k;
  if (g < 1 || g > P.k || i > g) return;
  const int64_t gu = (int64_t)b * (P.k + 1) + i;
  COSINE_TRACE_AT(P, 0);
  // this unit's C chunk records (every stats CTA is resident or done once this CTA runs)
  if ((threadIdx.x & 31) == 0) {
    uint32_t n;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(n) : "l"(P.ucnt + gu) : "memory");
      if ((int)n >= P.C) break;
      __nanosleep(100);
    }
  }
  __syncwarp();
  COSINE_TRACE_AT(P, 1);
  warp_decide<TT, TQ, kLogits>(P, b, i, g, s_gx[warp], s_tok[warp], &P.pdec[gu], true);
  COSINE_TRACE_AT(P, 2);
  if ((threadIdx.x & 31) == 0) {
    P.ucnt[gu] = 0;                 // ready for the next call
    red_release_add(&P.dcnt[b], 1);  // the decision before its count
  }
}

// One warp: the crossing chunk of t = u Q for a draw from the fused q = sum_n w_n q_n of record
// unit `rec` (SAMPLE selection, reading #3; u = U(rid, node, FUSE)).  The chunk masses come from
// the statistics pass's records: chunk r holds sum_n (w_n / sigma_n) dsum_{n,r} (LOGITS drafts:
// rescaled from the chunk max to the row max).  Lane 0 writes the kWFuseQ decision and the
// chunk's group range [g0, g1) with the target tc = t - (mass before the chunk) (reading #10;
// rounding past the total: the last positive chunk with tc = +inf).
template <bool kLogits>
__device__ __forceinline__ void chunk_crossing_warp(const SplitParams& P, int64_t rec, uint32_t node, uint64_t rid,
                                                    const double* s_w, const double* s_sig, const float* s_dmax,
                                                    Decision* s_d, int64_t* s_g0, int64_t* s_g1, double* s_tc,
                                                    double* s_Q) {
  const int lane = threadIdx.x & 31;
  const int N = P.N, C = P.C;
  const double k2 = (double)P.k2f;
  double m = 0.0;
  if (lane < C) {
    const PartRec* pr = P.parts + rec * C + lane;
    for (int n = 0; n < N; ++n) {
      const double ds = __ldcg(&pr->dsum[n]);
      double sc = 1.0;
      if (kLogits) sc = exp2((double)__ldcg(&pr->dmax[n]) * k2 - (double)s_dmax[n] * k2);
      if (ds != 0.0) m += (s_w[n] / s_sig[n]) * ds * sc;
    }
  }
  double incl = m;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double nb = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += nb;
  }
  const double Q = __shfl_sync(0xffffffffu, incl, 31);
  const double u = philox_u24(P.seed, rid, node, P.step, kTagFuse);
  const double t = u * Q;
  const unsigned hit = __ballot_sync(0xffffffffu, lane < C && m > 0.0 && incl > t);
  const unsigned pos = __ballot_sync(0xffffffffu, lane < C && m > 0.0);
  int r;
  double tc;
  if (hit) {
    r = __ffs(hit) - 1;
    tc = t - (__shfl_sync(0xffffffffu, incl, r) - __shfl_sync(0xffffffffu, m, r));
  } else {
    r = pos ? 31 - __clz(pos) : 0;
    tc = INFINITY;
  }
  if (lane == 0) {
    *s_g0 = (int64_t)r * P.cg;
    *s_g1 = min(P.ngroups, *s_g0 + P.cg);
    *s_tc = tc;
    *s_Q = Q;
    Decision d;
    d.need = 1;
    d.kind = kWFuseQ;
    d.xstar = -1;
    d.node = node;
    d.u = u;
    d.M = 0.f;
    d.invS = 0.f;
    d.k2 = P.k2f;
    for (int n = 0; n < kMaxN; ++n) {
      d.a[n] = (n < N) ? (float)(s_w[n] / s_sig[n]) : 0.f;
      d.dm[n] = (n < N) ? s_dmax[n] : 0.f;
    }
    *s_d = d;
  }
}

// Kernel B1 for SAMPLE selection (reading #3: x*_i ~ the fused q_i, the distribution-exact
// fusion; "direct ensemble sampling"): one CTA per unit, a programmatic dependent
// of stats_kernel that waits for its unit's C chunk records.
//  1. warp 0 combines the records (M, S, sigma) and the own-token gathers: confidences and the
//     fusion weights w (Eq. 4 weights; warp_decide_core stopped before x*);
//  2. the chunk masses of q come free from the statistics pass: chunk r holds
//     sum_n (w_n / sigma_n) dsum_{n,r} (rescaled to the row max for LOGITS drafts); the crossing
//     chunk of t = u Q, u = U(rid, i+1, FUSE), is found in one warp prefix over the C chunks;
//  3. the CTA scans only that chunk (block scan, reading #10) for x*, gathers o(x*), q_m(x*) and
//     takes the acceptance test u' q(x*) < o(x*).
// One chunk of the unit's N drafter rows (1/C of them) is re-read: the draw costs no full pass.
template <typename TT, typename TQ, bool kLogits, int NMAX>
__global__ void __launch_bounds__(kThreads) sample_decide_kernel(const SplitParams P) {
  __shared__ float s_gx[(kMaxN + 1) * kMaxN];
  __shared__ int32_t s_tok[kMaxN];
  __shared__ PosDec s_pd;
  __shared__ Decision s_d;
  __shared__ double s_w[kMaxN], s_sig[kMaxN];
  __shared__ float s_dmax[kMaxN];
  __shared__ double s_scan[kWarps];
  __shared__ int64_t s_wi[kWarps];
  __shared__ int64_t s_found, s_g0, s_g1;
  __shared__ float s_margin;
  __shared__ double s_tc, s_Q;
  __shared__ int s_go;
  const int tid = threadIdx.x, lane = tid & 31;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t unit = blockIdx.x;
  if (unit >= (int64_t)P.B * (P.k + 1)) return;
  const int b = (int)(unit / (P.k + 1)), i = (int)(unit % (P.k + 1));
  const int g = P.draft_len ? P.draft_len[b] : P.k;
  if (g < 1 || g > P.k || i > g) return;
  const int64_t gu = (int64_t)b * (P.k + 1) + i;
  const int N = P.N, C = P.C;
  const bool has_d = i < g;
  const double k2 = (double)P.k2f;
  const TQ* drow = (const TQ*)P.draft + ((int64_t)b * P.k + i) * N * P.ld_q;
  const TT* trow = (const TT*)P.target + gu * P.ld_t;
  if (tid == 0) {  // this unit's C chunk records (every stats CTA is resident or done by now)
    uint32_t n;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(n) : "l"(P.ucnt + gu) : "memory");
      if ((int)n >= C) break;
      __nanosleep(100);
    }
  }
  __syncthreads();
  if (tid < 32) {
    const UnitStats st = warp_combine<TT, TQ, kLogits>(P, b, i, has_d, true, s_gx, s_tok);
    warp_decide_core<kLogits>(P, b, i, has_d, st, s_gx, s_tok, &s_pd, false, s_w, s_sig, s_dmax);
    if (lane == 0) s_go = (has_d && s_pd.status == 0) ? 1 : 0;
    __syncwarp();
    if (s_go) chunk_crossing_warp<kLogits>(P, gu, (uint32_t)(i + 1), P.rids[b], s_w, s_sig, s_dmax, &s_d, &s_g0, &s_g1,
                                           &s_tc, &s_Q);
  }
  __syncthreads();
  if (s_go) {
    const int64_t y = scan_range<TT, TQ, kLogits, NMAX>(P, s_d, kWFuseQ, trow, drow, N, s_g0, s_g1, s_tc, s_Q,
                                                        s_scan, s_wi, &s_found, &s_margin);
    if (tid == 0) {
      PosDec& pd = s_pd;
      pd.xstar = (int32_t)y;
      if (y >= 0) {
        double q = 0.0;
        for (int m = 0; m < N; ++m) {
          const double dv = (double)load_one(drow + (int64_t)m * P.ld_q, y);
          q += s_w[m] * (kLogits ? exp2(dv * k2 - (double)s_dmax[m] * k2) / s_sig[m] : dv / s_sig[m]);
        }
        pd.qx = q;
        pd.u = philox_u24(P.seed, P.rids[b], (uint32_t)(i + 1), P.step, kTagAccept);
        // acceptance u * q(x*) < o(x*), i.e. u < min(1, o/q)
        pd.px = exp2((double)load_one(trow, y) * k2 - (double)pd.M * k2) / pd.S;
        pd.accept = (pd.u * pd.qx < pd.px);
        pd.m_fa = fmin_(fmin_(pd.m_fa, s_margin), (float)fabs(pd.u - pd.px / pd.qx));
      } else {
        pd.status = COSINE_REQ_EMPTY_ROW;  // unreachable: q has mass (every w_n, sigma_n > 0)
      }
    }
  }
  if (tid == 0) {
    P.pdec[gu] = s_pd;
    write_pos_debug(P, b, i, has_d, s_pd);
    P.ucnt[gu] = 0;                 // ready for the next call
    red_release_add(&P.dcnt[b], 1);  // the decision before its count
  }
}

// Kernel B1 for SAMPLE selection over probability drafts: one WARP per unit.  Steps 1-2 as
// sample_decide_kernel; the crossing chunk's 32-group slice sums, written by the statistics pass
// (stats_kernel<..., kSlices>), locate the slice of t in one more warp prefix (slice masses
// sum_n (w_n / sigma_n) slice_{n,s}), and one 32-lane scan of that slice (reading #10) finds x*.
// Re-reads 32 groups of the N drafter rows per unit instead of half a chunk.  A t that falls in
// no slice (the row's partial last group, or rounding at the chunk end) scans the whole chunk.
template <typename TT, typename TQ, int NMAX>
__global__ void __launch_bounds__(kThreads) sample_decide_w_kernel(const SplitParams P) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float s_gx[kWarps][(kMaxN + 1) * kMaxN];
  __shared__ int32_t s_tok[kWarps][kMaxN];
  __shared__ PosDec s_pd[kWarps];
  __shared__ Decision s_d[kWarps];
  __shared__ double s_w[kWarps][kMaxN], s_sig[kWarps][kMaxN];
  __shared__ float s_dmax[kWarps][kMaxN];
  __shared__ int64_t s_g0[kWarps], s_g1[kWarps];
  __shared__ double s_tc[kWarps], s_Q[kWarps];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t unit = (int64_t)blockIdx.x * kWarps + warp;
  if (unit >= (int64_t)P.B * (P.k + 1)) return;
  const int b = (int)(unit / (P.k + 1)), i = (int)(unit % (P.k + 1));
  const int g = P.draft_len ? P.draft_len[b] : P.k;
  if (g < 1 || g > P.k || i > g) return;
  const int64_t gu = (int64_t)b * (P.k + 1) + i;
  const int N = P.N, C = P.C;
  const bool has_d = i < g;
  const double k2 = (double)P.k2f;
  const TQ* drow = (const TQ*)P.draft + ((int64_t)b * P.k + i) * N * P.ld_q;
  const TT* trow = (const TT*)P.target + gu * P.ld_t;
  if (lane == 0) {  // this unit's C chunk records
    uint32_t n;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(n) : "l"(P.ucnt + gu) : "memory");
      if ((int)n >= C) break;
      __nanosleep(100);
    }
  }
  __syncwarp();
  const UnitStats st = warp_combine<TT, TQ, false>(P, b, i, has_d, true, s_gx[warp], s_tok[warp]);
  warp_decide_core<false>(P, b, i, has_d, st, s_gx[warp], s_tok[warp], &s_pd[warp], false, s_w[warp], s_sig[warp],
                          s_dmax[warp]);
  const int go = (has_d && s_pd[warp].status == 0) ? 1 : 0;
  if (go) {
    chunk_crossing_warp<false>(P, gu, (uint32_t)(i + 1), P.rids[b], s_w[warp], s_sig[warp], s_dmax[warp],
                               &s_d[warp], &s_g0[warp], &s_g1[warp], &s_tc[warp], &s_Q[warp]);
    __syncwarp();
    const Decision d = s_d[warp];
    const int64_t g0 = s_g0[warp], g1 = s_g1[warp];
    const double tc = s_tc[warp], Q = s_Q[warp];
    // ---- the slice of t within the chunk ----
    const int64_t r = g0 / P.cg;
    const int64_t gfe = min(g1, P.gfull);
    const int nsl = gfe > g0 ? (int)((gfe - g0 + kSliceGroups - 1) / kSliceGroups) : 0;
    const float* sl = P.slices + (gu * C + r) * P.nsl * N;
    double a[kMaxN];
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) a[n] = (n < N) ? s_w[warp][n] / s_sig[warp][n] : 0.0;
    int hs = -1;
    double tcs = 0.0, base = 0.0;
    for (int s0 = 0; s0 < nsl && hs < 0; s0 += 32) {
      const int s = s0 + lane;
      double m = 0.0;
      if (s < nsl)
#pragma unroll
        for (int n = 0; n < NMAX; ++n)
          if (n < N) m += a[n] * (double)__ldcg(&sl[(int64_t)s * N + n]);
      double incl = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double nb = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nb;
      }
      const double excl = base + incl - m;
      const unsigned hit = __ballot_sync(0xffffffffu, s < nsl && m > 0.0 && excl <= tc && tc < excl + m);
      if (hit) {
        const int src = __ffs(hit) - 1;
        hs = s0 + src;
        tcs = tc - __shfl_sync(0xffffffffu, excl, src);
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
    float margin = 0.f;
    int64_t y;
    if (hs >= 0) {
      const int64_t sb = g0 + (int64_t)kSliceGroups * hs;
      y = warp_scan_range<TT, TQ, false, NMAX>(P, d, kWFuseQ, trow, drow, N, sb, min(gfe, sb + kSliceGroups), tcs, Q,
                                               &margin);
    } else {
      y = warp_scan_range<TT, TQ, false, NMAX>(P, d, kWFuseQ, trow, drow, N, g0, g1, tc, Q, &margin);
    }
    if (lane == 0) {
      PosDec& p = s_pd[warp];
      p.xstar = (int32_t)y;
      if (y >= 0) {
        double q = 0.0;
        for (int m = 0; m < N; ++m)
          q += s_w[warp][m] * ((double)load_one(drow + (int64_t)m * P.ld_q, y) / s_sig[warp][m]);
        p.qx = q;
        p.u = philox_u24(P.seed, P.rids[b], (uint32_t)(i + 1), P.step, kTagAccept);
        // acceptance u * q(x*) < o(x*), i.e. u < min(1, o/q)
        p.px = exp2((double)load_one(trow, y) * k2 - (double)p.M * k2) / p.S;
        p.accept = (p.u * p.qx < p.px);
        p.m_fa = fmin_(fmin_(p.m_fa, margin), (float)fabs(p.u - p.px / p.qx));
      } else {
        p.status = COSINE_REQ_EMPTY_ROW;  // unreachable: q has mass (every w_n, sigma_n > 0)
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    P.pdec[gu] = s_pd[warp];
    write_pos_debug(P, b, i, has_d, s_pd[warp]);
    P.ucnt[gu] = 0;                 // ready for the next call
    red_release_add(&P.dcnt[b], 1);  // the decision before its count
  }
}

// ============================== cosine_fuse_drafts ==============================
// Eq. 4 token fusion alone (Alg. 1 TokenFusion P:376-381) on the split kernels:
// stats_kernel (P.mode = kSplitFuse: unit (b, i < k), the N drafter rows) -> fuse_decide_kernel
// (CTA per unit: sigma, confidences, weights, x* = X_{n*} or x* ~ q) -> [fuse_write_q_kernel]
// -> fuse_finish_kernel (per-request status: the first erroring position voids the request).
template <typename TT, typename TQ, bool kLogits, int NMAX>
__global__ void __launch_bounds__(kThreads) fuse_decide_kernel(const SplitParams P) {
  __shared__ float s_gx[(kMaxN + 1) * kMaxN];
  __shared__ int32_t s_tok[kMaxN];
  __shared__ PosDec s_pd;
  __shared__ Decision s_d;
  __shared__ double s_w[kMaxN], s_sig[kMaxN];
  __shared__ float s_dmax[kMaxN];
  __shared__ double s_scan[kWarps];
  __shared__ int64_t s_wi[kWarps];
  __shared__ int64_t s_found, s_g0, s_g1;
  __shared__ float s_margin;
  __shared__ double s_tc, s_Q;
  __shared__ int s_go;
  const int tid = threadIdx.x, lane = tid & 31;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // stats_kernel's records (PDL)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t unit = blockIdx.x;  // b * k + i
  if (unit >= (int64_t)P.B * P.k) return;
  const int b = (int)(unit / P.k), i = (int)(unit % P.k);
  const int N = P.N;
  const TQ* drow = (const TQ*)P.draft + unit * N * P.ld_q;
  if (tid < 32) {
    const UnitStats st = warp_combine<TT, TQ, kLogits>(P, b, i, true, true, s_gx, s_tok, false);
    warp_decide_core<kLogits>(P, b, i, true, st, s_gx, s_tok, &s_pd, false, s_w, s_sig, s_dmax);
    if (lane == 0) s_go = (s_pd.status == 0 && P.select == COSINE_SEL_SAMPLE) ? 1 : 0;
    __syncwarp();
    if (s_go) chunk_crossing_warp<kLogits>(P, unit, (uint32_t)(i + 1), P.rids[b], s_w, s_sig, s_dmax, &s_d, &s_g0,
                                           &s_g1, &s_tc, &s_Q);
  }
  __syncthreads();
  if (s_go) {  // SAMPLE: x* ~ q, scanned in its crossing chunk (reading #10)
    const int64_t y = scan_range<TT, TQ, kLogits, NMAX>(P, s_d, kWFuseQ, reinterpret_cast<const TT*>(drow), drow, N,
                                                        s_g0, s_g1, s_tc, s_Q, s_scan, s_wi, &s_found, &s_margin);
    if (tid == 0) {
      s_pd.xstar = (int32_t)y;
      s_pd.m_fa = fmin_(s_pd.m_fa, s_margin);
      if (y < 0) s_pd.status = COSINE_REQ_EMPTY_ROW;  // unreachable: q has mass
    }
  }
  if (tid == 0) {
    const PosDec& pd = s_pd;
    P.pdec[unit] = pd;  // status, x*, margin, a = w / sigma (fuse_write_q_kernel, fuse_finish_kernel)
    P.fuse_tokens[unit] = pd.status ? -1 : pd.xstar;
    for (int n = 0; n < N; ++n) {
      if (P.fuse_w) P.fuse_w[unit * N + n] = pd.status ? NAN : pd.w[n];
      if (P.fuse_sig) P.fuse_sig[unit * N + n] = pd.status ? NAN : pd.sig[n];
    }
  }
}

// The fused distribution q_i(v) = sum_n w_n d_n(v) / sigma_n (POINT: delta_{x*}) into
// fused_q [B][k][ld_fq] fp32: CTA (unit, chunk), one group per thread per step.
template <typename TT, typename TQ, bool kLogits, int NMAX>
__global__ void __launch_bounds__(kThreads) fuse_write_q_kernel(const SplitParams P) {
  __shared__ PosDec s_pd;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // fuse_decide_kernel's decisions (PDL)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t unit = blockIdx.x / P.C;
  const int rank = (int)(blockIdx.x % P.C);
  const int N = P.N;
  if (threadIdx.x == 0) s_pd = P.pdec[unit];
  __syncthreads();
  if (s_pd.status) return;
  Decision d;
  d.k2 = P.k2f;
  for (int n = 0; n < kMaxN; ++n) {
    d.a[n] = s_pd.a[n];
    d.dm[n] = s_pd.dm[n];
  }
  const TQ* drow = (const TQ*)P.draft + unit * N * P.ld_q;
  float* qrow = P.fused_q + unit * P.ld_fq;
  const int64_t gb = (int64_t)rank * P.cg, ge = min(P.ngroups, gb + P.cg);
  for (int64_t gi = gb + threadIdx.x; gi < ge; gi += kThreads) {
    float w[8];
    if (P.weight_mode == COSINE_W_POINT) {
#pragma unroll
      for (int e = 0; e < 8; ++e) w[e] = (gi * kGroup + e == (int64_t)s_pd.xstar) ? 1.f : 0.f;
    } else {
      group_weights<TT, TQ, kLogits, NMAX>(P, d, kWWriteQ, reinterpret_cast<const TT*>(drow), drow, N, gi, w);
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
}

// Per request: the first erroring position's status voids every fused token (as the oracle
// does); otherwise INFO_NEAR_TIE when a decision margin is < 1e-6 (reading #18).
__global__ void __launch_bounds__(kThreads) fuse_finish_kernel(const SplitParams P);

// ============================== cosine_sample_residual ==============================
// The final-token draw alone on the split kernels: stats_kernel (mode kSplitSample:
// unit b = request b's row, + its N drafter rows for the residual's validity checks) ->
// sample_prep_kernel (warp per request: the row statistics — or the caller's M, S — and the
// caller's weights / normalisers as the request's two position records: position 0 "rejected"
// (residual, g = 1) or accepted (bonus)) -> resample_kernel (the tile masses and the scan).
template <typename TT, typename TQ>
__global__ void __launch_bounds__(kThreads) sample_prep_kernel(const SplitParams P) {
  __shared__ float s_gx[kWarps][(kMaxN + 1) * kMaxN];
  __shared__ int32_t s_tok[kWarps][kMaxN];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // stats_kernel's records (PDL)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int b = blockIdx.x * kWarps + warp;
  if (b >= P.B) return;
  const int N = P.N;
  const bool has_d = P.draft != nullptr;
  const bool greedy = P.greedy != 0;
  // the records of unit b: combine as warp_combine does (no gathers)
  const PartRec* parts = P.parts + (int64_t)b * P.C;
  const bool own = lane < P.C;
  const double k2 = (double)P.k2f;
  const float tmax = own ? __ldcg(&parts[lane].tmax) : kNegBig;
  const int bad = __reduce_or_sync(0xffffffffu, own ? __ldcg(&parts[lane].bad) : 0);
  float M = 0.f;
  double S = 0.0;
  int64_t amax = -1;
  bool t_nf = false, t_empty = false, d_nf = false;
  if (greedy) {
    float bv = own ? tmax : -INFINITY;
    int64_t bi = own ? (int64_t)__ldcg((const long long*)&parts[lane].targ) : -1;
    warp_argmax(bv, bi);
    t_nf = (bad & 1) != 0;
    t_empty = bi < 0;
    amax = bi;
    M = bv;
  } else {
    M = warp_max(tmax);
    const double tsum = own ? __ldcg(&parts[lane].tsum) : 0.0;
    S = warp_sum(tsum != 0.0 ? tsum * exp2((double)tmax * k2 - (double)M * k2) : 0.0);
    // NaN / +inf anywhere in the row makes the (recomputed) sum non-finite
    t_nf = !isfinite(S) || !isfinite(M);
    t_empty = !t_nf && !(S > 0.0);
  }
  if (has_d) {
    if (bad & 2) d_nf = true;
    for (int n = 0; n < N; ++n) {
      const double sv = warp_sum(own ? __ldcg(&parts[lane].dsum[n]) : 0.0);
      if (!isfinite(sv)) d_nf = true;
    }
  }
  (void)s_gx;
  (void)s_tok;
  if (lane != 0) return;
  int st = 0;
  if (!greedy && P.row_max) {  // the caller's statistics (M = max l, S = sum exp((l - M) / T))
    M = P.row_max[b];
    S = (double)P.row_sumexp[b];
    t_empty = !t_nf && !(S > 0.0 && isfinite(S) && isfinite(M));
  }
  if (t_nf) st = COSINE_REQ_NONFINITE_INPUT;
  else if (t_empty) st = COSINE_REQ_EMPTY_ROW;
  if (!st && !greedy && has_d) {
    if (d_nf) st = COSINE_REQ_NONFINITE_INPUT;
    for (int n = 0; n < N && !st; ++n) {
      const float nv = P.norm_in[(int64_t)b * N + n];
      if (!(nv > 0.f) || !isfinite(nv)) st = COSINE_REQ_EMPTY_ROW;
    }
  }
  PosDec pd;
  init_posdec(pd);
  pd.status = st;
  pd.M = M;
  pd.S = S;
  pd.amax = amax;
  pd.m_fa = INFINITY;
  for (int n = 0; n < N; ++n) {
    pd.a[n] = has_d ? (float)((double)P.w_in[(int64_t)b * N + n] / (double)P.norm_in[(int64_t)b * N + n]) : 0.f;
    pd.dm[n] = 0.f;
  }
  // position 0 rejected -> the residual of position 0 (L = 0 < g = 1); accepted -> the bonus (L = g)
  pd.accept = has_d ? 0 : 1;
  PosDec* out = P.pdec + (int64_t)b * 2;
  out[0] = pd;
  pd.status = 0;
  out[1] = pd;
}

// Lazy round r (NEXT-1): one warp per request still verifying decides position r (as
// decide_kernel), then stops the request at its first rejection / error / bonus row.  The
// positions after the stop are never read; their decision slots are written as "accepted, OK"
// so that the request view of resample_kernel sees L and the errors of positions <= L only.
template <typename TT, typename TQ, bool kLogits>
__global__ void __launch_bounds__(kThreads) lazy_decide_kernel(const SplitParams P) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x * kWarps + warp;
  __shared__ float s_gx[kWarps][(kMaxN + 1) * kMaxN];
  __shared__ int32_t s_tok[kWarps][kMaxN];
  if (!P.fused) asm volatile("griddepcontrol.wait;" ::: "memory");  // this round's records (PDL)
  if (b >= P.B) return;
  const int r0 = P.lazy - 1;
  const int g = P.draft_len ? P.draft_len[b] : P.k;
  if (g < 1 || g > P.k || r0 > g) return;
  if (r0 > 0 && P.lz[b] != 0) return;
  PosDec* pds = P.pdec + (int64_t)b * (P.k + 1);
  const int r1 = min(g, r0 + P.lazy_span - 1);
  // fused: wait for each position's C chunk records (device counters; every stats CTA of the
  // round is resident or done once this CTA runs), consume and reset every counted position
  auto wait_unit = [&](int r) {
    if (!P.fused) return;
    if (lane == 0) {
      const int32_t* cnt = P.ucnt + (int64_t)b * (P.k + 1) + r;
      uint32_t n;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(n) : "l"(cnt) : "memory");
        if ((int)n >= P.C) break;
        __nanosleep(100);
      }
    }
    __syncwarp();
  };
  bool stop = false;
  for (int r = r0; r <= r1 && !stop; ++r) {  // the round's positions in order
    wait_unit(r);
    warp_decide<TT, TQ, kLogits>(P, b, r, g, s_gx[warp], s_tok[warp], &pds[r], true);
    __syncwarp();
    int st = 0;
    if (lane == 0) {
      const PosDec& pd = pds[r];
      st = (pd.status != 0 || r == g || !pd.accept) ? 1 : 0;
      if (st) {
        PosDec ok;
        init_posdec(ok);
        for (int j = r + 1; j <= g; ++j) pds[j] = ok;
      }
    }
    stop = __shfl_sync(0xffffffffu, st, 0) != 0;
  }
  if (P.fused) {  // the round's streamed positions: all counted -> reset for the next round / call
    for (int r = r0; r <= r1; ++r) wait_unit(r);
    if (lane == 0)
      for (int r = r0; r <= r1; ++r) P.ucnt[(int64_t)b * (P.k + 1) + r] = 0;
  }
  if (lane == 0) P.lz[b] = stop ? -1 : 0;
}

// The request-level view of the position decisions (first error, first rejection L, margins).
struct ReqView {
  int32_t g, err, L, sample;  // sample: T > 0 and no error -> a final inverse-CDF draw at row L
  float tm;
};
__device__ __forceinline__ ReqView request_view(const SplitParams& P, const PosDec* pds, int g) {
  ReqView v;
  v.g = g;
  v.err = 0;
  v.L = g;
  v.tm = INFINITY;
  for (int j = 0; j <= g; ++j)
    if (!v.err && pds[j].status) v.err = pds[j].status;
  for (int j = 0; j < g; ++j)
    if (!pds[j].accept) { v.L = j; break; }
  for (int j = 0; j <= v.L; ++j) v.tm = fmin_(v.tm, pds[j].m_fa);
  v.sample = (!v.err && !P.greedy) ? 1 : 0;
  return v;
}

// The same view computed by one warp from global memory (lanes over positions; every lane
// returns it): the first error, the first rejection L, the smallest margin on positions <= L.
__device__ __forceinline__ ReqView request_view_warp(const SplitParams& P, const PosDec* pds, int g) {
  const int lane = threadIdx.x & 31;
  ReqView v;
  v.g = g;
  v.err = 0;
  v.L = g;
  v.tm = INFINITY;
  for (int j0 = 0; j0 <= g; j0 += 32) {
    const int j = j0 + lane;
    const bool in = j <= g;
    const int st = in ? pds[j].status : 0;
    const int acc = in ? pds[j].accept : 1;
    const unsigned e = __ballot_sync(0xffffffffu, st != 0);
    if (!v.err && e) v.err = __shfl_sync(0xffffffffu, st, __ffs(e) - 1);
    const unsigned r = __ballot_sync(0xffffffffu, j < g && !acc);
    if (v.L == g && r) v.L = j0 + __ffs(r) - 1;
  }
  float tm = INFINITY;
  for (int j = lane; j <= v.L; j += 32) tm = fmin_(tm, pds[j].m_fa);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tm = fmin_(tm, __shfl_xor_sync(0xffffffffu, tm, o));
  v.tm = tm;
  v.sample = (!v.err && !P.greedy) ? 1 : 0;
  return v;
}

__device__ __forceinline__ Decision sample_decision(const SplitParams& P, int b, const PosDec& pl,
                                                    const ReqView& v) {
  const uint64_t rid = P.rids[b];
  const bool resid = v.L < v.g;
  Decision d;
  d.need = 1;
  d.kind = resid ? ((P.weight_mode == COSINE_W_POINT) ? kWPoint : kWResidual) : kWBonus;
  d.xstar = pl.xstar - (int32_t)P.v0;  // local column (vocabulary-sharded mode)
  // Philox node of the draw: L (reading #19); cosine_sample_residual: the caller's node id
  d.node = (P.mode == kSplitSample) ? P.node_ids[b] : (uint32_t)v.L;
  d.u = philox_u24(P.seed, rid, d.node, P.step, kTagSample);
  d.M = pl.M;
  d.invS = (float)(1.0 / pl.S);
  d.k2 = P.k2f;
  for (int n = 0; n < kMaxN; ++n) { d.a[n] = pl.a[n]; d.dm[n] = pl.dm[n]; }
  return d;
}

// Raw (1 + N) row groups of one vocabulary group, loaded before any arithmetic so that every
// load of an iteration is in flight together (the weights are computed afterwards).
template <typename TT, typename TQ, int NMAX>
struct RowGroups {
  Group<TT> t;
  Group<TQ> d[NMAX];
  __device__ __forceinline__ void zero() {
    t.zero();
#pragma unroll
    for (int n = 0; n < NMAX; ++n) d[n].zero();
  }
  // Every member is assigned on every path (zeros when not needed): a member left unset on
  // one path forces the whole array into local memory.
  __device__ __forceinline__ void load(const TT* trow, const TQ* drow, int64_t ld_q, int Nd, bool need_t,
                                       bool need_q, int64_t gi) {
    if (need_t) t.load(trow, gi);
    else t.zero();
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      if (need_q && n < Nd) d[n].load(drow + (int64_t)n * ld_q, gi);
      else d[n].zero();
    }
  }
};

// Sampling weights of a FULL group from already-loaded rows (same arithmetic as group_weights).
template <typename TT, typename TQ, bool kLogits, int NMAX>
__device__ __forceinline__ float group_mass(const RowGroups<TT, TQ, NMAX>& rg, const Decision& d, int kind,
                                            int Nd, int64_t gi) {
  float q[8], t[8], w[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) q[e] = 0.f;
  const bool need_q = (kind == kWResidual);
  if (need_q) {
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      if (n < Nd) {
        float f[8];
        rg.d[n].unpack(f);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float qv = kLogits ? ex2((f[e] - d.dm[n]) * d.k2) : f[e];
          q[e] = fmaf(d.a[n], qv, q[e]);
        }
      }
    }
  }
  rg.t.unpack(t);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float pe = ex2((t[e] - d.M) * d.k2);
    float x;
    if (kind == kWBonus) {
      x = pe;
    } else {
      const float p = pe * d.invS;
      if (kind == kWResidual) x = fmaxf(p - q[e], 0.f);
      else if (kind == kWPoint) x = (gi * kGroup + e == (int64_t)d.xstar) ? fmaxf(p - 1.f, 0.f) : p;
      else x = p;  // kWProb
    }
    w[e] = x;
  }
  return sum8(w);
}


// One warp: Z = sum of the tile masses seg[0 .. nseg) in a fixed order (lane l owns a contiguous
// run of tiles, then a warp scan), and the crossing tile of t = u * Z: the smallest s with
// O_s + seg[s] > t (O_s = the masses before s) and tc = t - O_s.  If rounding leaves no crossing
// in the owning lane's run, tstar = that run's last positive tile with tc = +inf (the scan then
// takes the tile's last positive entry, reading #10).  All lanes return Z; lane 0 tstar / tc.
template <bool kGlobal>
__device__ __forceinline__ double warp_tile_crossing(const double* seg, int64_t nseg, double u,
                                                     int64_t* tstar, double* tc, double t_abs = -1.0) {
  const int lane = threadIdx.x & 31;
  auto at = [&](int64_t s2) { return kGlobal ? __ldcg(seg + s2) : seg[s2]; };
  const int64_t per = (nseg + 31) / 32;
  const int64_t s0 = min(nseg, lane * per), s1 = min(nseg, s0 + per);
  double part = 0.0;
  for (int64_t s2 = s0; s2 < s1; ++s2) part += at(s2);
  double incl = part;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double nb = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += nb;
  }
  const double Z = __shfl_sync(0xffffffffu, incl, 31);
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.0;
  const double t = (t_abs >= 0.0) ? t_abs : u * Z;  // t_abs: an absolute target (sharded mode)
  const unsigned m = __ballot_sync(0xffffffffu, Z > 0.0 && incl > t && s1 > s0);
  int64_t ts = -1;
  double c = 0.0;
  if (m) {
    const int f = __ffs(m) - 1;
    if (lane == f) {
      double O = excl;
      int64_t lastpos = -1;
      for (int64_t s2 = s0; s2 < s1; ++s2) {
        const double z = at(s2);
        if (z > 0.0) lastpos = s2;
        if (O + z > t) { ts = s2; c = t - O; break; }
        O += z;
      }
      if (ts < 0) { ts = lastpos; c = INFINITY; }
    }
    ts = __shfl_sync(0xffffffffu, ts, f);
    c = __shfl_sync(0xffffffffu, c, f);
  }
  *tstar = ts;
  *tc = c;
  return Z;
}

// The local mass of request b's final draw in vocabulary-sharded mode: into this rank's send
// slot (NCCL all-gather) or straight into every rank's gather buffer + one arrival on each
// (p2p; cosine_shard.cuh).  One thread.
__device__ __forceinline__ void shard_z_out(const SplitParams& P, int b, double z) {
  if (!P.p2p) {
    P.zsend[b] = z;
    return;
  }
  for (int g = 0; g < P.G; ++g) P.z_peer[g][b] = z;
  __threadfence_system();
  for (int g = 0; g < P.G; ++g) atomicAdd_system(P.cnt_peer[g] + 1, 1ull);
}

// The final draw of a request, split in parts of kSegTilesPerCta 2048-entry tiles:
//  1. the request's position decisions give the first rejection L (request_view);
//  2. each part streams its tiles of the (1+N) rows at L (or the bonus row) — same group
//     mapping as the statistics pass, one tile of loads per thread in flight — and writes each
//     tile's residual (or bonus) mass;
//  3. the LAST part of the request (device-scope counter) sums the tile masses in tile order,
//     finds the crossing tile, scans it block-wide (reading #10) and writes the outputs.
constexpr int kSegTilesPerCta = 8;

struct ResampleSmem {
  PosDec pd[kMaxPos];
  ReqView v;
  Decision d;
  double red[kWarps][kSegTilesPerCta];
  double scan[kWarps];
  double seg[kMaxSeg];
  int64_t wi[kWarps];
  int64_t found, tstar;
  double tc, Z;
  float margin;
  int last, kind, deg;
};

// All threads: request b's decisions (positions 0..g) into shared memory, the request view and,
// when a final inverse-CDF draw is needed, its Decision.  Ends with a barrier.
__device__ __forceinline__ void load_request(const SplitParams& P, int b, int g, ResampleSmem& s) {
  const int tid = threadIdx.x;
  const int nw = (int)(sizeof(PosDec) / 4);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(P.pdec + (int64_t)b * (P.k + 1));
  uint32_t* dst = reinterpret_cast<uint32_t*>(s.pd);
  for (int w = tid; w < (g + 1) * nw; w += kThreads) dst[w] = __ldcg(src + w);  // L2 (other CTAs wrote them)
  __syncthreads();
  if (tid == 0) {
    const ReqView v = request_view(P, s.pd, g);
    s.v = v;
    if (v.sample) s.d = sample_decision(P, b, s.pd[v.L], v);
  }
  __syncthreads();
}

// Outputs of a request without a final draw: a per-request error, or greedy (y = argmax of
// row L, reading #7).  Threads of one CTA.
__device__ __forceinline__ void write_plain_outputs(const SplitParams& P, int b, const ResampleSmem& s) {
  const ReqView& v = s.v;
  if (P.mode == kSplitSample) {  // cosine_sample_residual: an error, or greedy (the row's argmax)
    if (threadIdx.x == 0) {
      P.out_token[b] = v.err ? -1 : (int32_t)s.pd[0].amax;
      P.status[b] = v.err;
    }
    return;
  }
  int32_t* out = P.out_tokens + (int64_t)b * (P.k + 1);
  for (int j = threadIdx.x; j <= P.k; j += kThreads)
    out[j] = v.err ? -1 : ((j < v.L) ? s.pd[j].xstar : (j == v.L ? (int32_t)s.pd[v.L].amax : -1));
  if (threadIdx.x == 0) {
    P.accept_len[b] = v.err ? -1 : v.L;
    P.status[b] = v.err ? v.err : ((v.tm < 1e-6f) ? COSINE_INFO_NEAR_TIE : 0);
    if (!v.err && P.dbg.tie_margin) P.dbg.tie_margin[b] = v.tm;
  }
}

__device__ __forceinline__ void write_bad_len(const SplitParams& P, int b) {
  int32_t* out = P.out_tokens + (int64_t)b * (P.k + 1);
  P.accept_len[b] = -1;
  for (int j = 0; j <= P.k; ++j) out[j] = -1;
  P.status[b] = COSINE_REQ_BAD_DRAFT_LEN;
}

// Part `part` of request b's final draw (s loaded by load_request, s.v.sample set).
template <typename TT, typename TQ, bool kLogits, int NMAX>
__device__ __forceinline__ void resample_tiles(const SplitParams& P, int b, int part, ResampleSmem& s) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const ReqView v = s.v;
  const Decision& d = s.d;
  const int kind0 = d.kind;
  const int Nd = (v.L < v.g) ? P.N : 0;
  const bool need_q = (kind0 == kWResidual);
  const bool smode = P.mode == kSplitSample;  // cosine_sample_residual: request b's own row group
  const TT* trow = (const TT*)P.target + (smode ? (int64_t)b : (int64_t)b * (P.k + 1) + v.L) * P.ld_t;
  const TQ* drow = (const TQ*)P.draft + (smode ? (int64_t)b : (int64_t)b * P.k + v.L) * P.N * P.ld_q;
  const int64_t tile0 = (int64_t)part * P.tpc;
  const int ntiles = (int)min((int64_t)P.tpc, P.nseg - tile0);
#pragma unroll 1
  for (int j = 0; j < ntiles; ++j) {  // one tile of (1+N) loads per thread in flight
    const int64_t g0 = (tile0 + j) * kTileGroups + tid;
    double m0 = 0.0;
    if (g0 < P.gfull) {
      RowGroups<TT, TQ, NMAX> r0;
      r0.load(trow, drow, P.ld_q, Nd, true, need_q, g0);
      m0 = (double)group_mass<TT, TQ, kLogits, NMAX>(r0, d, kind0, Nd, g0);
    } else if (g0 < P.ngroups) {  // the row's partial last group
      float w[8];
      group_weights<TT, TQ, kLogits, NMAX>(P, d, kind0, trow, drow, Nd, g0, w);
      m0 = (double)sum8(w);
    }
    m0 = warp_sum(m0);
    if (lane == 0) s.red[warp][j] = m0;
  }
  __syncthreads();
  if (tid < ntiles) {
    double z = 0.0;
    for (int w = 0; w < kWarps; ++w) z += s.red[w][tid];
    P.segsum[(int64_t)b * P.nseg + tile0 + tid] = z;
  }
  __syncthreads();
  if (tid == 0) {  // the masses before the count; the last part acquires the others'
    const int old = atom_acq_rel_add(&P.counters[b], 1);
    s.last = (old == P.spr - 1);
    if (s.last && P.fused) P.dcnt[b] = 0;  // every part of the request has passed its wait
  }
  __syncthreads();
  COSINE_TRACE_AT(P, 5);
  if (!s.last) return;
  // ---------------- the last part of the request: crossing tile, scan, outputs ----------------
  const double* ss = P.segsum + (int64_t)b * P.nseg;
  const bool in_smem = P.nseg <= kMaxSeg;
  if (in_smem)
    for (int64_t t = tid; t < P.nseg; t += kThreads) s.seg[t] = __ldcg(ss + t);
  __syncthreads();
  if (warp == 0) {
    int64_t tstar = -1;
    double tc = 0.0;
    const double Z = in_smem ? warp_tile_crossing<false>(s.seg, P.nseg, d.u, &tstar, &tc)
                             : warp_tile_crossing<true>(ss, P.nseg, d.u, &tstar, &tc);
    if (lane == 0) {
      P.counters[b] = 0;  // ready for the next call
      if (P.shard) {      // vocabulary-sharded: this rank's mass; shard_sample_kernel goes on
        shard_z_out(P, b, Z);
      } else {
        int kind = kind0, dg = 0;
        if (!(Z > 0.0) && (kind == kWResidual || kind == kWPoint)) {
          kind = kWProb;  // all mass cancelled: resample from o (reading #11)
          dg = 1;
          tstar = -1;
        }
        s.Z = Z;
        s.kind = kind;
        s.deg = dg;
        s.tstar = tstar;
        s.tc = tc;
      }
    }
  }
  if (P.shard) return;
  __syncthreads();
  const int kind = s.kind, deg = s.deg;
  double Z = s.Z;
  int64_t y = -1;
  float margin = INFINITY;
  if (deg) {  // rare: the whole row from o, block-wide
    double acc = 0.0;
    for (int64_t gi = tid; gi < P.ngroups; gi += kThreads) {
      float w[8];
      group_weights<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, gi, w);
      acc += (double)sum8(w);
    }
    Z = block_sum(acc, s.scan);
    if (tid == 0) s.Z = Z;
    __syncthreads();
    Z = s.Z;
    y = scan_range<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, 0, P.ngroups, d.u * Z, Z, s.scan,
                                          s.wi, &s.found, &s.margin);
    margin = s.margin;
  } else if (s.tstar >= 0) {
    COSINE_TRACE_AT(P, 6);
    const int64_t sb = s.tstar * kTileGroups;
    y = scan_range<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, sb, min(P.ngroups, sb + kTileGroups),
                                          s.tc, Z, s.scan, s.wi, &s.found, &s.margin);
    margin = s.margin;
  }
  if (smode) {
    if (tid == 0) {
      P.out_token[b] = (int32_t)y;
      P.status[b] = (deg ? COSINE_INFO_DEGENERATE_RESIDUAL : 0) | (margin < 1e-6f ? COSINE_INFO_NEAR_TIE : 0) |
                    (y < 0 ? 0xff : 0);
    }
    return;
  }
  int32_t* out = P.out_tokens + (int64_t)b * (P.k + 1);
  for (int j = tid; j <= P.k; j += kThreads) out[j] = (j < v.L) ? s.pd[j].xstar : (j == v.L ? (int32_t)y : -1);
  if (tid == 0) {
    P.accept_len[b] = v.L;
    const float tm = fmin_(v.tm, margin);
    P.status[b] = (deg ? COSINE_INFO_DEGENERATE_RESIDUAL : 0) | (tm < 1e-6f ? COSINE_INFO_NEAR_TIE : 0) |
                  (y < 0 ? 0xff : 0);
    if (P.dbg.residual_mass) P.dbg.residual_mass[b] = (float)((kind == kWBonus) ? Z * (double)d.invS : Z);
    if (P.dbg.tie_margin) P.dbg.tie_margin[b] = tm;
  }
}

// One item of kernel B2: part `part` of request b's final draw (the decisions are complete).
template <typename TT, typename TQ, bool kLogits, int NMAX>
__device__ __forceinline__ void resample_item(const SplitParams& P, int b, int part, int g, ResampleSmem& s) {
  if (g < 1 || g > P.k) {
    if (part == 0 && threadIdx.x == 0) {
      if (P.shard) shard_z_out(P, b, 0.0);  // the outputs come from shard_finish_kernel
      else write_bad_len(P, b);
    }
    return;
  }
  COSINE_TRACE_AT(P, 1);
  load_request(P, b, g, s);
  if (!s.v.sample) {
    if (P.fused && threadIdx.x == 0) {  // the request's last part resets the counters
      if (atomicAdd(&P.counters[b], 1) == P.spr - 1) {
        P.counters[b] = 0;
        P.dcnt[b] = 0;
      }
    }
    if (part == 0) {
      if (P.shard) {
        if (threadIdx.x == 0) shard_z_out(P, b, 0.0);
      } else {
        write_plain_outputs(P, b, s);
      }
    }
    return;
  }
  resample_tiles<TT, TQ, kLogits, NMAX>(P, b, part, s);
}

// Kernel B2: CTA (request b, part), a programmatic dependent of the kernel that wrote the
// decisions.  Split path (P.fused): waits for its request's g + 1 decisions only (every
// decide_kernel CTA is resident or done once this CTA runs, so the wait always ends), not for
// the whole grid.  (Measured slower on c3 and not kept: a persistent one-wave grid taking the
// parts from a device counter, 462 vs 454 us; two tiles per thread in flight at 4 CTAs / SM,
// 465 us.)
template <typename TT, typename TQ, bool kLogits, int NMAX>
__global__ void __launch_bounds__(kThreads, 5) resample_kernel(const SplitParams P) {
  __shared__ __align__(16) ResampleSmem s;
  const int b = P.b_off + blockIdx.x / P.spr;  // spr = CTAs per request
  const int part = blockIdx.x % P.spr;
  const int g = P.draft_len ? P.draft_len[b] : P.k;
  COSINE_TRACE_AT(P, 0);
  if (P.fused) {
    if (g >= 1 && g <= P.k) {
      if (threadIdx.x == 0) {
        uint32_t n;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(n) : "l"(P.dcnt + b) : "memory");
          if ((int)n >= g + 1) break;
          __nanosleep(200);
        }
      }
      __syncthreads();
    }
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the decisions (PDL)
  }
  resample_item<TT, TQ, kLogits, NMAX>(P, b, part, g, s);
  COSINE_TRACE_AT(P, 7);
}

// ============================== small batches: one launch ==============================
// The three kernels' work in ONE cooperative launch for a batch whose (unit, chunk) grid is
// co-resident (c1, c2: latency-bound — the split path pays three dependent launches and a
// device round trip per hand-off).  CTA (unit u = (b, i), chunk r), p = i C + r its index among
// request b's (k + 1) C CTAs:
//  1. the chunk's statistics (stats_body) and its count on ucnt[u]; the unit's LAST chunk CTA
//     (the one whose count completes the unit, so no wait) decides the unit with one warp
//     (Eq. 4 fusion and acceptance, warp_decide) and counts the decision on dcnt[b];
//  2. CTAs p < spr are the parts of the request's final draw: wait for the request's g + 1
//     decisions (every CTA they wait for is resident: cooperative launch), then the tile
//     masses of row L and, in the last part, the crossing tile and its scan (resample_tiles).
template <typename TT, typename TQ, bool kLogits, int NMAX>
__global__ void __launch_bounds__(kThreads, 4) tiny_kernel(const SplitParams P) {
  __shared__ __align__(16) ResampleSmem s;
  __shared__ float s_gx[(kMaxN + 1) * kMaxN];
  __shared__ int32_t s_tok[kMaxN];
  __shared__ int s_decide;
  const int C = P.C;
  const int64_t u = blockIdx.x / C;
  const int r = (int)(blockIdx.x % C);
  const int b = (int)(u / (P.k + 1)), i = (int)(u % (P.k + 1));
  const int p = i * C + r;
  const int g = P.draft_len ? P.draft_len[b] : P.k;
  COSINE_TRACE_AT(P, 0);
  // (the one-row unrolled loop measured slower here: c2 56 vs 53 us)
  const int64_t gu = stats_body<TT, TQ, kLogits, NMAX, false, false>(P, u, r);
  __syncthreads();
  COSINE_TRACE_AT(P, 1);
  if (threadIdx.x == 0) {
    int last = 0;
    if (gu >= 0)  // the record before the count; the unit's last chunk acquires the others'
      last = atom_acq_rel_add(&P.ucnt[gu], 1) == C - 1;
    s_decide = last;
  }
  __syncthreads();
  if (s_decide && threadIdx.x < 32) {
    warp_decide<TT, TQ, kLogits>(P, b, i, g, s_gx, s_tok, &P.pdec[gu], true);
    if (threadIdx.x == 0) {
      P.ucnt[gu] = 0;                 // ready for the next call
      red_release_add(&P.dcnt[b], 1);  // the decision before its count
    }
    COSINE_TRACE_AT(P, 2);
  }
  if (p >= P.spr) return;
  if (g < 1 || g > P.k) {
    if (p == 0 && threadIdx.x == 0) write_bad_len(P, b);
    return;
  }
  if (threadIdx.x == 0) {
    uint32_t n;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(n) : "l"(P.dcnt + b) : "memory");
      if ((int)n >= g + 1) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
  COSINE_TRACE_AT(P, 3);
  load_request(P, b, g, s);
  COSINE_TRACE_AT(P, 4);
  if (!s.v.sample) {
    if (threadIdx.x == 0 && atomicAdd(&P.counters[b], 1) == P.spr - 1) {  // the last part resets
      P.counters[b] = 0;
      P.dcnt[b] = 0;
    }
    if (p == 0) write_plain_outputs(P, b, s);
    return;
  }
  resample_tiles<TT, TQ, kLogits, NMAX>(P, b, p, s);
  COSINE_TRACE_AT(P, 7);
}

}  // namespace cosine
