// cosine_shard.cuh — vocabulary-sharded verification (SURVEY §8(e) "Vocab" mode, config c5).
//
// Every rank holds the columns [v0, v0 + V) of every target and drafter row (the layout a
// tensor-parallel LM head produces) and calls cosine_verify_batch collectively.
// The rows never move; three small all-gathers carry what the decisions need:
//   1. stats_kernel (local columns) -> shard_pack_kernel: one record per (request, position):
//      local max / sum-exp of the target row, local drafter normalisers, local greedy argmax and
//      the candidate gathers l(X_n), d_m(X_n) of the tokens this rank owns  ->  all-gather.
//   2. shard_decide_kernel: every rank combines the G records IN RANK ORDER (fixed-order fp64
//      sums, so all ranks take bit-identical decisions: Eq. 4 fusion P:406-411, acceptance
//      P:130-131) and finds the first rejection L.
//   3. resample_kernel (shard mode): the local mass of the final draw's weights over this
//      rank's columns of row L (residual max(0, o - q), or the bonus row), per
//      256-group tile  ->  all-gather of the local masses Z_g.
//   4. shard_sample_kernel: the rank whose prefix interval [O_g, O_g + Z_g) holds t = u Z scans
//      its crossing tile (reading #10: ascending GLOBAL index, the concatenation of the shards
//      in rank order)  ->  all-gather of the owner's token;  shard_finish_kernel writes the
//      (replicated) outputs on every rank.
#pragma once

#include "cosine_split.cuh"

namespace cosine {

struct YRec {  // the final token as seen by one rank
  int32_t y;   // global token id (owner) or -1
  float margin;
  int32_t deg;
  float z;
};

// Record layout (32-bit words): 0 M (f32), 1 flags (bit0 target bad, bit1 drafter bad, bits
// 8.. own mask over n), 2 greedy argmax (global id, -1 none), 3 its value (f32), 4-5 S (f64),
// 6-7 pad, then sig f64[N], dmax f32[N], tx f32[N] = l(X_n), dx f32[N][N] = d_m(X_n) (m-major).
__host__ __device__ constexpr int shard_rec_words(int N) { return (8 + 2 * N + N + N + N * N + 3) & ~3; }
struct RecOff {
  int sig, dmax, tx, dx;
  __device__ __forceinline__ explicit RecOff(int N)
      : sig(8), dmax(8 + 2 * N), tx(8 + 3 * N), dx(8 + 4 * N) {}
};

constexpr int kMaxPeers = 8;  // ranks of an in-kernel (NVLink peer memory) exchange

// One thread: wait until this rank's arrival counter x reaches the call's target (every rank's
// contribution to exchange x is in this rank's gather buffer).  Gives up after ~5 s (a rank that
// never arrives must not hang the GPU: the outputs are then wrong, not stuck).
__device__ __forceinline__ void p2p_wait(const SplitParams& P, int x) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long n;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(n) : "l"(P.cnt_own + x) : "memory");
    if (n >= P.tgt[x]) break;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 5000000000ull) break;
    __nanosleep(64);
  }
}
// One thread: this thread's writes into the peers' buffers before one arrival on each of them.
__device__ __forceinline__ void p2p_arrive(const SplitParams& P, int x) {
  __threadfence_system();
  for (int g = 0; g < P.G; ++g) atomicAdd_system(P.cnt_peer[g] + x, 1ull);
}
__device__ __forceinline__ void shard_put_y(const SplitParams& P, int b, const YRec& y) {
  if (!P.p2p) {
    P.ysend[b] = y;
    return;
  }
  for (int g = 0; g < P.G; ++g) P.y_peer[g][b] = y;
  p2p_arrive(P, 2);
}

// ---------------- 1. the local record of a unit (one warp per unit) ----------------
template <typename TT, typename TQ, bool kLogits>
__device__ __forceinline__ void shard_pack_unit(const SplitParams& P, int64_t unit, int b, int i, int g) {
  const int lane = threadIdx.x & 31;
  const bool has_d = i < g;
  const int N = P.N, C = P.C;
  const double k2 = (double)P.k2f;
  const RecOff ro(N);
  uint32_t* rec = P.rec_send + unit * P.rec_words;
  float* recf = reinterpret_cast<float*>(rec);
  // gathers of the candidates this rank owns (lane = m * N + n)
  bool mine = false;
  if (has_d && lane < N * (N + 1)) {
    const int n = lane % N, m = lane / N;
    const int32_t tk = P.draft_tokens[((int64_t)b * P.k + i) * N + n];
    mine = tk >= (int64_t)P.v0 && (int64_t)tk < P.v0 + P.V;
    float v = 0.f;
    if (mine) {
      const int64_t lv = (int64_t)tk - P.v0;
      if (m < N) v = load_one((const TQ*)P.draft + (((int64_t)b * P.k + i) * N + m) * P.ld_q, lv);
      else v = load_one((const TT*)P.target + ((int64_t)b * (P.k + 1) + i) * P.ld_t, lv);
    }
    if (m < N) recf[ro.dx + m * N + n] = v;
    else recf[ro.tx + n] = v;
  }
  const uint32_t ownmask = __ballot_sync(0xffffffffu, mine && lane < N) & ((1u << N) - 1u);
  // combine this rank's chunk records (chunk r in lane r), as warp_decide does
  const PartRec* parts = P.parts + unit * C;
  const bool own = lane < C;
  const float tmax = own ? __ldcg(&parts[lane].tmax) : kNegBig;
  const int bad = __reduce_or_sync(0xffffffffu, own ? __ldcg(&parts[lane].bad) : 0);
  float M = kNegBig, bv = -INFINITY;
  double S = 0.0;
  int64_t bi = -1;
  if (P.greedy) {
    bv = own ? tmax : -INFINITY;
    bi = own ? (int64_t)__ldcg((const long long*)&parts[lane].targ) : -1;
    warp_argmax(bv, bi);
  } else {
    M = warp_max(tmax);
    const double tsum = own ? __ldcg(&parts[lane].tsum) : 0.0;
    S = warp_sum(tsum != 0.0 ? tsum * exp2((double)tmax * k2 - (double)M * k2) : 0.0);
  }
  double sig[kMaxN];
  float dmx[kMaxN];
  for (int n = 0; n < N; ++n) {
    sig[n] = 0.0;
    dmx[n] = kNegBig;
    if (!has_d) continue;
    const double ds = own ? __ldcg(&parts[lane].dsum[n]) : 0.0;
    if (kLogits) {
      const float dmr = own ? __ldcg(&parts[lane].dmax[n]) : kNegBig;
      dmx[n] = warp_max(dmr);
      sig[n] = warp_sum(ds != 0.0 ? ds * exp2((double)dmr * k2 - (double)dmx[n] * k2) : 0.0);
    } else {
      sig[n] = warp_sum(ds);
    }
  }
  if (lane == 0) {
    recf[0] = P.greedy ? bv : M;
    rec[1] = (uint32_t)(bad & 3) | (ownmask << 8);
    rec[2] = (uint32_t)(int32_t)(bi >= 0 ? bi + P.v0 : -1);
    recf[3] = bv;
    *reinterpret_cast<double*>(rec + 4) = S;
    double* sg = reinterpret_cast<double*>(rec + ro.sig);
    for (int n = 0; n < N; ++n) {
      sg[n] = sig[n];
      recf[ro.dmax + n] = dmx[n];
    }
    if (!has_d)
      for (int n = 0; n < N; ++n) recf[ro.tx + n] = 0.f;
  }
  if (P.p2p) {  // the record into every rank's gather buffer (rank-major, as the all-gather's)
    __syncwarp();
    for (int gg = 0; gg < P.G; ++gg) {
      uint32_t* dst = P.rec_peer[gg] + unit * P.rec_words;
      for (int w = lane; w < P.rec_words; w += 32) dst[w] = rec[w];
    }
  }
}

template <typename TT, typename TQ, bool kLogits>
__global__ void __launch_bounds__(kThreads) shard_pack_kernel(const SplitParams P) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t unit = (int64_t)blockIdx.x * kWarps + warp;
  if (!P.ucount) asm volatile("griddepcontrol.wait;" ::: "memory");  // stats_kernel's records (PDL)
  const int b = (int)(unit / (P.k + 1)), i = (int)(unit % (P.k + 1));
  const bool valid = unit < (int64_t)P.B * (P.k + 1);
  const int g = valid ? (P.draft_len ? P.draft_len[b] : P.k) : 0;
  if (valid && g >= 1 && g <= P.k && i <= g) {
    if (P.ucount) {  // this unit's C chunk records (every stats CTA is resident or done by now)
      if (lane == 0) {
        uint32_t n;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(n) : "l"(P.ucnt + unit) : "memory");
          if ((int)n >= P.C) break;
          __nanosleep(100);
        }
        P.ucnt[unit] = 0;  // ready for the next call (nothing else reads it)
      }
      __syncwarp();
    }
    shard_pack_unit<TT, TQ, kLogits>(P, unit, b, i, g);
  }
  if (P.p2p) {  // every rank's copy of this CTA's records, then one arrival per CTA on every rank
    __syncthreads();
    if (threadIdx.x == 0) p2p_arrive(P, 0);
  }
}

// ---------------- 2. global decisions from the G records (one warp per unit) ----------------
template <bool kLogits>
__global__ void __launch_bounds__(kThreads) shard_decide_kernel(const SplitParams P) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t unit = (int64_t)blockIdx.x * kWarps + warp;
  __shared__ float s_gx[kWarps][(kMaxN + 1) * kMaxN];
  __shared__ int32_t s_tok[kWarps][kMaxN];
  if (P.p2p) {  // every rank's records have arrived
    if (tid == 0) p2p_wait(P, 0);
    __syncthreads();
  }
  const int64_t units = (int64_t)P.B * (P.k + 1);
  if (unit >= units) return;
  const int b = (int)(unit / (P.k + 1)), i = (int)(unit % (P.k + 1));
  const int g = P.draft_len ? P.draft_len[b] : P.k;
  if (g < 1 || g > P.k || i > g) return;
  const bool has_d = i < g;
  const int N = P.N, G = P.G;
  const double k2 = (double)P.k2f;
  const RecOff ro(N);
  const bool own = lane < G;  // lane r reads rank r's record
  const uint32_t* rec = P.rec_all + ((int64_t)(own ? lane : 0) * units + unit) * P.rec_words;
  const float* recf = reinterpret_cast<const float*>(rec);
  const uint32_t flags = own ? rec[1] : 0u;
  const int bad = (int)__reduce_or_sync(0xffffffffu, flags & 3u);
  UnitStats st;
  st.M = 0.f;
  st.S = 0.0;
  st.amax = -1;
  st.t_nf = st.t_empty = st.d_nf = st.d_empty = st.tok_bad = false;
  st.sig = NAN;
  st.dmx = kNegBig;
  if (P.greedy) {
    float bv = own ? recf[3] : -INFINITY;
    int64_t bi = own ? (int64_t)(int32_t)rec[2] : -1;
    warp_argmax(bv, bi);  // best value, lowest global index on ties (reading #5 / #7)
    st.t_nf = (bad & 1) != 0;
    st.t_empty = bi < 0;
    st.amax = bi;
    st.M = bv;
  } else {
    const float Mr = own ? recf[0] : kNegBig;
    st.M = warp_max(Mr);
    const double Sr = own ? *reinterpret_cast<const double*>(rec + 4) : 0.0;
    st.S = warp_sum(Sr != 0.0 ? Sr * exp2((double)Mr * k2 - (double)st.M * k2) : 0.0);
    st.t_nf = !isfinite(st.S) || !isfinite(st.M);
    st.t_empty = !st.t_nf && !(st.S > 0.0);
  }
  bool tok_bad = false;
  if (has_d) {
    if (bad & 2) st.d_nf = true;
    const double* sg = reinterpret_cast<const double*>(rec + ro.sig);
    for (int n = 0; n < N; ++n) {
      const double ds = own ? sg[n] : 0.0;
      double sv;
      float mx = kNegBig;
      if (kLogits) {
        const float dmr = own ? recf[ro.dmax + n] : kNegBig;
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
    // the candidate gathers come from the rank that owns each token (lane n: candidate n)
    for (int n = 0; n < N; ++n) {
      const unsigned owners = __ballot_sync(0xffffffffu, own && ((flags >> (8 + n)) & 1u));
      const int src = owners ? __ffs(owners) - 1 : -1;
      if (lane == n) {
        const int32_t tk = P.draft_tokens[((int64_t)b * P.k + i) * N + n];
        s_tok[warp][n] = tk;
        if (src < 0 || tk < 0 || (int64_t)tk >= P.Vg) {
          tok_bad = true;
        } else {
          const float* rs = reinterpret_cast<const float*>(P.rec_all + ((int64_t)src * units + unit) * P.rec_words);
          for (int m = 0; m < N; ++m) s_gx[warp][m * kMaxN + n] = rs[ro.dx + m * N + n];
          s_gx[warp][N * kMaxN + n] = rs[ro.tx + n];
        }
      }
    }
  }
  st.tok_bad = __any_sync(0xffffffffu, tok_bad);
  __syncwarp();
  warp_decide_core<kLogits>(P, b, i, has_d, st, s_gx[warp], s_tok[warp], &P.pdec[unit], true);
}

// ---------------- 4. the owner of t scans its crossing tile (one CTA per request) ----------------
template <typename TT, typename TQ, bool kLogits, int NMAX>
__global__ void __launch_bounds__(kThreads) shard_sample_kernel(const SplitParams P) {
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  __shared__ __align__(16) PosDec s_pd[kMaxPos];
  __shared__ ReqView s_v;
  __shared__ Decision s_d;
  __shared__ double s_scan[kWarps];
  __shared__ int64_t s_wi[kWarps];
  __shared__ int64_t s_found;
  __shared__ float s_margin;
  __shared__ int s_owner, s_fb, s_kind, s_deg;
  __shared__ double s_tc, s_Z;
  __shared__ int64_t s_tstar;
  YRec yr;
  yr.y = -1;
  yr.margin = INFINITY;
  yr.deg = 0;
  yr.z = 0.f;
  if (P.p2p) {  // every rank's local masses have arrived
    if (tid == 0) p2p_wait(P, 1);
    __syncthreads();
  }
  const int g = P.draft_len ? P.draft_len[b] : P.k;
  if (g < 1 || g > P.k) {
    if (tid == 0) shard_put_y(P, b, yr);
    return;
  }
  {
    const int nw = (int)(sizeof(PosDec) / 4);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(P.pdec + (int64_t)b * (P.k + 1));
    uint32_t* dst = reinterpret_cast<uint32_t*>(s_pd);
    for (int w = tid; w < (g + 1) * nw; w += kThreads) dst[w] = src[w];
  }
  __syncthreads();
  if (tid == 0) {
    const ReqView v = request_view(P, s_pd, g);
    s_v = v;
    if (v.sample) s_d = sample_decision(P, b, s_pd[v.L], v);
  }
  __syncthreads();
  const ReqView v = s_v;
  if (!v.sample) {
    if (tid == 0) shard_put_y(P, b, yr);
    return;
  }
  const Decision d = s_d;
  const int Nd = (v.L < v.g) ? P.N : 0;
  const TT* trow = (const TT*)P.target + ((int64_t)b * (P.k + 1) + v.L) * P.ld_t;
  const TQ* drow = (const TQ*)P.draft + ((int64_t)b * P.k + v.L) * P.N * P.ld_q;
  if (tid == 0) {
    // the global mass of the final draw is the rank-ordered sum of the local masses
    double zr[32];
    int kind = d.kind, deg = 0;
    double Z = 0.0;
    for (int r = 0; r < P.G; ++r) { zr[r] = P.zall[(int64_t)r * P.B + b]; Z += zr[r]; }
    if (!(Z > 0.0) && (kind == kWResidual || kind == kWPoint)) {
      // all mass cancelled: resample from o (reading #11); o's local masses follow from
      // the step-1 records of row L: S_g 2^((M_g - M) k2) / S
      kind = kWProb;
      deg = 1;
      const int64_t units = (int64_t)P.B * (P.k + 1);
      const int64_t unit = (int64_t)b * (P.k + 1) + v.L;
      const double k2 = (double)P.k2f;
      const PosDec& pl = s_pd[v.L];
      Z = 0.0;
      for (int r = 0; r < P.G; ++r) {
        const uint32_t* rec = P.rec_all + ((int64_t)r * units + unit) * P.rec_words;
        const float Mr = reinterpret_cast<const float*>(rec)[0];
        const double Sr = *reinterpret_cast<const double*>(rec + 4);
        zr[r] = (Sr != 0.0) ? Sr * exp2((double)Mr * k2 - (double)pl.M * k2) / pl.S : 0.0;
        Z += zr[r];
      }
    }
    const double t = d.u * Z;
    int owner = -1, fb = 0;
    double O = 0.0, Oown = 0.0;
    for (int r = 0; r < P.G && Z > 0.0; ++r) {
      if (zr[r] > 0.0 && O <= t && t < O + zr[r]) { owner = r; Oown = O; break; }
      O += zr[r];
    }
    if (owner < 0 && Z > 0.0) {  // rounding: the last positive entry overall (reading #10)
      for (int r = P.G - 1; r >= 0; --r)
        if (zr[r] > 0.0) { owner = r; fb = 1; break; }
    }
    s_owner = owner;
    s_fb = fb;
    s_kind = kind;
    s_deg = deg;
    s_Z = Z;
    s_tc = t - Oown;
    s_tstar = -1;
    if (owner == P.rank && !deg && fb) {  // rounding past the total: the last positive tile
      const double* ss = P.segsum + (int64_t)b * P.nseg;
      for (int64_t s2 = P.nseg - 1; s2 >= 0; --s2)
        if (__ldcg(ss + s2) > 0.0) { s_tstar = s2; break; }
      s_tc = INFINITY;
    }
  }
  __syncthreads();
  if (s_owner == P.rank && !s_deg && !s_fb && threadIdx.x < 32) {  // this rank's crossing tile
    int64_t ts;
    double tc;
    warp_tile_crossing<true>(P.segsum + (int64_t)b * P.nseg, P.nseg, 0.0, &ts, &tc, s_tc);
    if (threadIdx.x == 0) {
      s_tstar = ts;
      s_tc = (ts >= 0) ? tc : INFINITY;
    }
  }
  __syncthreads();
  if (s_owner == P.rank) {
    const int kind = s_kind;
    const double Z = s_Z;
    int64_t y = -1;
    if (s_deg) {
      y = scan_range<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, 0, P.ngroups, s_fb ? INFINITY : s_tc, Z,
                                            s_scan, s_wi, &s_found, &s_margin);
    } else if (s_tstar >= 0) {
      const int64_t sb = s_tstar * kTileGroups;
      y = scan_range<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, sb, min(P.ngroups, sb + kTileGroups), s_tc,
                                            Z, s_scan, s_wi, &s_found, &s_margin);
    }
    if (tid == 0) {
      yr.y = (y >= 0) ? (int32_t)(y + P.v0) : -1;
      yr.margin = (y >= 0) ? s_margin : 0.f;
    }
  }
  __syncthreads();  // (p2p: every read of this rank's gather buffers precedes the last arrival)
  if (tid == 0) {
    yr.deg = s_deg;
    yr.z = (float)s_Z;
    shard_put_y(P, b, yr);
  }
}

#ifndef COSINE_DTYPE_TU  // non-template kernel: defined in the host TU only

// ---------------- 5. the replicated outputs (one thread per request) ----------------
__global__ void __launch_bounds__(kThreads) shard_finish_kernel(const SplitParams P) {
  // one warp per request: lanes over its positions (a thread per request walked them serially)
  if (P.p2p) {  // every rank's token has arrived
    if (threadIdx.x == 0) p2p_wait(P, 2);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (b >= P.B) return;
  const int g = P.draft_len ? P.draft_len[b] : P.k;
  int32_t* out = P.out_tokens + (int64_t)b * (P.k + 1);
  if (g < 1 || g > P.k) {
    for (int j = lane; j <= P.k; j += 32) out[j] = -1;
    if (lane == 0) {
      P.accept_len[b] = -1;
      P.status[b] = COSINE_REQ_BAD_DRAFT_LEN;
    }
    return;
  }
  const PosDec* pds = P.pdec + (int64_t)b * (P.k + 1);
  const ReqView v = request_view_warp(P, pds, g);
  if (!v.sample) {
    for (int j = lane; j <= P.k; j += 32)
      out[j] = v.err ? -1 : ((j < v.L) ? pds[j].xstar : (j == v.L ? (int32_t)pds[v.L].amax : -1));
    if (lane == 0) {
      P.accept_len[b] = v.err ? -1 : v.L;
      P.status[b] = v.err ? v.err : ((v.tm < 1e-6f) ? COSINE_INFO_NEAR_TIE : 0);
      if (!v.err && P.dbg.tie_margin) P.dbg.tie_margin[b] = v.tm;
    }
    return;
  }
  // the owner's token: the first rank (in rank order) with y >= 0; rank 0's deg / z otherwise
  YRec mine;
  mine.y = -1;
  mine.margin = 0.f;
  mine.deg = 0;
  mine.z = 0.f;
  if (lane < P.G) mine = P.yall[(int64_t)lane * P.B + b];
  const unsigned has = __ballot_sync(0xffffffffu, lane < P.G && mine.y >= 0);
  const int src = has ? __ffs(has) - 1 : 0;
  YRec yr;
  yr.y = __shfl_sync(0xffffffffu, mine.y, src);
  yr.margin = __shfl_sync(0xffffffffu, mine.margin, src);
  yr.deg = __shfl_sync(0xffffffffu, mine.deg, src);
  yr.z = __shfl_sync(0xffffffffu, mine.z, src);
  if (!has) yr.y = -1, yr.margin = 0.f;
  for (int j = lane; j <= P.k; j += 32) out[j] = (j < v.L) ? pds[j].xstar : (j == v.L ? yr.y : -1);
  if (lane == 0) {
    P.accept_len[b] = v.L;
    const float tm = fmin_(v.tm, yr.margin);
    P.status[b] = (yr.deg ? COSINE_INFO_DEGENERATE_RESIDUAL : 0) | (tm < 1e-6f ? COSINE_INFO_NEAR_TIE : 0) |
                  (yr.y < 0 ? 0xff : 0);
    const bool bonus = !yr.deg && v.L == v.g;
    if (P.dbg.residual_mass) P.dbg.residual_mass[b] = bonus ? (float)((double)yr.z / pds[v.L].S) : yr.z;
    if (P.dbg.tie_margin) P.dbg.tie_margin[b] = tm;
  }
}

#endif

}  // namespace cosine
