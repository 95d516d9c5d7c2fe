// cosine_stream.cuh — the persistent, warp-specialised sm_100a kernel behind
// cosine_verify_batch (Eq. 4 ARGMAX fusion, T > 0 or greedy).
//
// Layout of the work:
//   * a thread-block cluster of C CTAs owns a static list of requests (b = cluster id,
//     + ncl, ...) and walks each request's positions i = 0..gamma_b in order; CTA r of the
//     cluster owns vocabulary chunk r of every row;
//   * warp 8 of each CTA is a TMA producer: one elected lane issues 1-D bulk copies
//     (cp.async.bulk, SASS UBLKCP) of 2048-element row tiles (the target row and the N
//     drafter rows of the unit) into a ring of smem stages guarded by full / empty mbarriers,
//     running ahead across position and request boundaries so HBM never waits on the
//     consumers' reductions or decisions;
//   * warps 0-7 (256 consumer threads) reduce each tile (online max / sum-exp of the target
//     logits, drafter row sums) and, at the end of a position, push a 200-byte record into
//     every CTA of the cluster over DSMEM (remote mbarrier arrive, release.cluster);
//   * every CTA combines the C records in rank order and takes the SAME decisions (fusion,
//     acceptance, first rejection), so no decision has to be broadcast.  The first rejection
//     of a request (or its bonus row) triggers one cooperative inverse-CDF round over the
//     rows just streamed, which are L2-resident: pass A (chunk sums, exchanged over DSMEM),
//     pass B (tile scan of the crossing chunk only);
//   * CTA 0 writes the request's outputs; no global atomics, one launch per call.
#pragma once

namespace cosine {

constexpr int kConsWarps = 8;
constexpr int kConsThreads = kConsWarps * 32;   // 256
constexpr int kProdWarp = kConsWarps;            // warp 8: TMA producer
constexpr int kDecWarp = kConsWarps + 1;         // warp 9: decisions + sampling
constexpr int kStreamThreads = kConsThreads + 64;
constexpr int kRecSlots = 6;                     // record ring (units in flight per cluster)
constexpr int kMaxCS = 8;                        // max cluster size of the persistent kernel
constexpr int kTileGroups = kConsThreads;        // one 8-element group per consumer thread
constexpr int kTileElems = kTileGroups * kGroup; // 2048
constexpr int kMaxStages = 12;

struct StreamParams {
  int B, k, N;
  int64_t V, ld_t, ld_q, ngroups, gfull;
  int C, ncl;
  int64_t cgroups;     // groups per CTA chunk
  int stages;
  int t_slot, q_slot;  // bytes per row slot in a stage
  int stage_bytes;
  float k2f;
  double k2d;
  int greedy, weight_mode;
  int debug_flags;  // bit0: skip sampling rounds (profiling only; results invalid)
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
};

__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cta(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Non-blocking probe of an mbarrier phase (acquire, cluster scope).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_cta(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Blocking waits with a watchdog: a protocol bug traps (~4 s) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity) {
  if (mbar_try_cluster(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_cluster(bar, parity))
    if (clock64() - t0 > (1LL << 33)) __trap();
}
__device__ __forceinline__ void mbar_wait_ring(uint64_t* bar, uint32_t parity) {
  if (mbar_try_cta(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_cta(bar, parity))
    if (clock64() - t0 > (1LL << 33)) __trap();
}
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <typename T>
__device__ __forceinline__ void smem_group(const unsigned char* slot, int idx, float f[8]);
template <>
__device__ __forceinline__ void smem_group<__nv_bfloat16>(const unsigned char* slot, int idx, float f[8]) {
  const uint4 a = reinterpret_cast<const uint4*>(slot)[idx];
  f[0] = __uint_as_float(a.x << 16); f[1] = __uint_as_float(a.x & 0xffff0000u);
  f[2] = __uint_as_float(a.y << 16); f[3] = __uint_as_float(a.y & 0xffff0000u);
  f[4] = __uint_as_float(a.z << 16); f[5] = __uint_as_float(a.z & 0xffff0000u);
  f[6] = __uint_as_float(a.w << 16); f[7] = __uint_as_float(a.w & 0xffff0000u);
}
template <>
__device__ __forceinline__ void smem_group<float>(const unsigned char* slot, int idx, float f[8]) {
  const float4 a = reinterpret_cast<const float4*>(slot)[2 * idx];
  const float4 b = reinterpret_cast<const float4*>(slot)[2 * idx + 1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// Decisions of one position, identical in every CTA of the cluster.
struct UnitDec {
  int32_t status, accept, xstar, need, kind;
  uint32_t node;
  double u_s;
  int64_t amax;
  float Mf, m_fa;
  double M, S, px, qx, u;
  double sig[kMaxN], c[kMaxN], w[kMaxN];
  float dmax[kMaxN];
};

// Sampling work the decision warp posts to its own consumer warps (run at their next position
// boundary, so the consumers never wait on another CTA).
enum JobType : int { kJobSum = 0, kJobScan = 1 };
constexpr int kJobSlots = 8;
struct Job {
  int32_t type, b, i, kind, deg;
  uint32_t zcount;  // sampling-exchange counter (selects the s_z buffer)
  double tc, Z;
  Decision d;
};

// Combine the C records (rank order = ascending vocabulary) and decide position i of request b.
template <bool kLogits>
__device__ __noinline__ void decide_unit(const StreamParams& P, const CtaRec* recs, int C,
                                         const float (*gx)[kMaxN], const int32_t* tok, bool has_d,
                                         int i, int g, uint64_t rid, int first_rej, UnitDec& o) {
  const int N = P.N;
  const bool greedy = P.greedy != 0;
  o.status = 0; o.accept = 1; o.xstar = -1; o.need = 0; o.kind = kWBonus; o.node = 0; o.u_s = 0.0;
  o.amax = -1; o.Mf = 0.f; o.m_fa = INFINITY; o.M = 0.0; o.S = 0.0; o.px = o.qx = o.u = NAN;
  bool t_nf = false, t_empty = false, d_nf = false, d_empty = false, tok_bad = false, zero = false;
  if (greedy) {
    float bv = -INFINITY;
    int64_t bi = -1;
    int bad = 0;
    for (int r = 0; r < C; ++r) {
      bad |= recs[r].bad;
      if (recs[r].targ >= 0 && (bi < 0 || recs[r].tmax > bv)) { bv = recs[r].tmax; bi = recs[r].targ; }
    }
    t_nf = (bad & 1) != 0;
    t_empty = (bi < 0);
    o.amax = bi;
    o.Mf = bv;
    o.M = bv;
  } else {
    float M = kNegBig;
    for (int r = 0; r < C; ++r) M = fmaxf(M, recs[r].tmax);
    double S = 0.0;
    for (int r = 0; r < C; ++r)
      if (recs[r].tsum != 0.0) S += recs[r].tsum * exp2(((double)recs[r].tmax - (double)M) * P.k2d);
    o.Mf = M;
    o.M = M;
    o.S = S;
    t_nf = !isfinite(S) || !isfinite(M);
    t_empty = !t_nf && !(S > 0.0);
  }
  if (has_d) {
    int bad = 0;
    for (int r = 0; r < C; ++r) bad |= recs[r].bad;
    if (bad & 2) d_nf = true;
    for (int n = 0; n < N; ++n) {
      double s = 0.0;
      float mx = kNegBig;
      if (kLogits) {
        for (int r = 0; r < C; ++r) mx = fmaxf(mx, recs[r].dmax[n]);
        for (int r = 0; r < C; ++r)
          if (recs[r].dsum[n] != 0.0) s += recs[r].dsum[n] * exp2(((double)recs[r].dmax[n] - (double)mx) * P.k2d);
        if (!isfinite(mx)) d_nf = true;
      } else {
        for (int r = 0; r < C; ++r) s += recs[r].dsum[n];
      }
      o.sig[n] = s;
      o.dmax[n] = mx;
      if (!isfinite(s)) d_nf = true;
      else if (!(s > 0.0)) d_empty = true;
    }
    for (int n = 0; n < N; ++n)
      if (tok[n] < 0 || (int64_t)tok[n] >= P.V) tok_bad = true;
  }
  int stc = 0;
  if (tok_bad) stc = COSINE_REQ_TOKEN_OUT_OF_RANGE;
  else if (t_nf || d_nf) stc = COSINE_REQ_NONFINITE_INPUT;
  else if (t_empty || d_empty) stc = COSINE_REQ_EMPTY_ROW;
  if (!stc && has_d) {
    for (int n = 0; n < N; ++n) {
      const double dv = (double)gx[n][n];
      o.c[n] = kLogits ? exp2((dv - (double)o.dmax[n]) * P.k2d) / o.sig[n] : dv / o.sig[n];
      if (o.c[n] == 0.0) zero = true;
    }
    if (zero) stc = COSINE_REQ_ZERO_PROB_DRAFT;
  }
  o.status = stc;
  if (stc) return;
  if (has_d) {
    // Eq. 4: n* = argmax_n c_n, ties -> lowest n; fused weights (reading #2)
    int ns = 0;
    for (int n = 1; n < N; ++n)
      if (o.c[n] > o.c[ns]) ns = n;
    double second = -1.0;
    for (int n = 0; n < N; ++n)
      if (n != ns && o.c[n] > second) second = o.c[n];
    o.m_fa = (N > 1) ? (float)((o.c[ns] - second) / o.c[ns]) : INFINITY;
    if (P.weight_mode == COSINE_W_CONF) {
      double sc = 0.0;
      for (int n = 0; n < N; ++n) sc += o.c[n];
      for (int n = 0; n < N; ++n) o.w[n] = o.c[n] / sc;
    } else if (P.weight_mode == COSINE_W_UNIFORM) {
      for (int n = 0; n < N; ++n) o.w[n] = 1.0 / (double)N;
    } else {
      for (int n = 0; n < N; ++n) o.w[n] = (n == ns) ? 1.0 : 0.0;
    }
    o.xstar = tok[ns];
    if (P.weight_mode == COSINE_W_POINT) {
      o.qx = 1.0;
    } else {
      double q = 0.0;
      for (int m = 0; m < N; ++m) {
        const double dv = (double)gx[m][ns];
        const double qm = kLogits ? exp2((dv - (double)o.dmax[m]) * P.k2d) / o.sig[m] : dv / o.sig[m];
        q += o.w[m] * qm;
      }
      o.qx = q;
    }
    o.u = philox_u24(P.seed, rid, (uint32_t)(i + 1), P.step, kTagAccept);
    if (greedy) {
      o.accept = ((int64_t)o.xstar == o.amax);
    } else {
      // acceptance u * q(x*) < o(x*), i.e. u < min(1, o/q)
      o.px = exp2(((double)gx[N][ns] - o.M) * P.k2d) / o.S;
      o.accept = (o.u * o.qx < o.px);
      o.m_fa = fmin_(o.m_fa, (float)fabs(o.u - o.px / o.qx));
      if (!o.accept && first_rej == g) {  // the first rejection: resample
        o.need = 1;
        o.kind = (P.weight_mode == COSINE_W_POINT) ? kWPoint : kWResidual;
        o.node = (uint32_t)i;
        o.u_s = philox_u24(P.seed, rid, (uint32_t)i, P.step, kTagSample);
      }
    }
  } else if (!greedy && first_rej == g) {  // every draft accepted: bonus
    o.need = 1;
    o.kind = kWBonus;
    o.node = (uint32_t)g;
    o.u_s = philox_u24(P.seed, rid, (uint32_t)g, P.step, kTagSample);
  }
}


template <typename TT, typename TQ, bool kLogits, int NMAX>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_kernel(const StreamParams P) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = P.C;
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x / C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = P.N;

  extern __shared__ __align__(128) unsigned char s_ring[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t empty_bar[kMaxStages];
  __shared__ __align__(8) uint64_t rec_full[kRecSlots];
  __shared__ __align__(8) uint64_t rec_free[kRecSlots];
  __shared__ __align__(8) uint64_t z_bar[2];
  __shared__ __align__(8) uint64_t y_bar;
  __shared__ CtaRec s_rec[kRecSlots][kMaxCS];
  __shared__ float s_gx[kRecSlots][kMaxN + 1][kMaxN];
  __shared__ int32_t s_tok[kRecSlots][kMaxN];
  __shared__ double s_z[2][kMaxCS];
  __shared__ SampleOut s_y;
  __shared__ Decision s_dec;
  __shared__ UnitDec s_ud;
  __shared__ float s_wf[kWarps][1 + kMaxN];
  __shared__ float s_wv[kWarps];
  __shared__ int64_t s_wi[kWarps];
  __shared__ double s_wd[kWarps][1 + kMaxN];
  __shared__ int32_t s_wbad[kWarps];
  __shared__ double s_scan[kWarps];
  __shared__ int64_t s_found;
  __shared__ float s_margin;
  __shared__ Job s_job[kJobSlots];
  __shared__ volatile int32_t s_posted, s_dec_done;
  __shared__ int32_t s_nready, s_final;

  if (tid == 0) {
    s_posted = 0;
    s_dec_done = 0;
    for (int s = 0; s < P.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kConsWarps);
    }
    for (int s = 0; s < kRecSlots; ++s) {
      mbar_init(&rec_full[s], (uint32_t)C);
      mbar_init(&rec_free[s], (uint32_t)C);
    }
    mbar_init(&z_bar[0], (uint32_t)C);
    mbar_init(&z_bar[1], (uint32_t)C);
    mbar_init(&y_bar, 1);
    fence_mbar_init_cluster();
  }
  cluster.sync();

  const int64_t cb = (int64_t)rank * P.cgroups;  // this CTA's chunk [cb, ce) in groups
  const int64_t ce = min(P.ngroups, cb + P.cgroups);
  const int ntiles = ce > cb ? (int)((ce - cb + kTileGroups - 1) / kTileGroups) : 0;
  const int tsz = sizeof(TT), qsz = sizeof(TQ);
  const bool greedy = P.greedy != 0;

  if (warp == kProdWarp) {
    // =============================== TMA producer ===============================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int b = cid; b < P.B; b += P.ncl) {
        const int g = P.draft_len ? P.draft_len[b] : P.k;
        if (g < 1 || g > P.k) continue;
        for (int i = 0; i <= g; ++i) {
          const int nrows = 1 + (i < g ? N : 0);
          const unsigned char* trow = (const unsigned char*)P.target + ((int64_t)b * (P.k + 1) + i) * P.ld_t * tsz;
          const unsigned char* drow = (const unsigned char*)P.draft + ((int64_t)b * P.k + i) * N * P.ld_q * qsz;
          for (int t = 0; t < ntiles; ++t) {
            const int64_t g0 = cb + (int64_t)t * kTileGroups;
            const int64_t g1 = min(ce, g0 + kTileGroups);
            const int64_t e0 = g0 * kGroup, e1 = min(P.V, g1 * kGroup);
            const uint32_t tb = (uint32_t)(((e1 - e0) * tsz + 15) & ~15LL);
            const uint32_t qb = (uint32_t)(((e1 - e0) * qsz + 15) & ~15LL);
            mbar_wait_ring(&empty_bar[stage], phase ^ 1u);
            mbar_expect_tx(&full_bar[stage], tb + (uint32_t)(nrows - 1) * qb);
            unsigned char* st = s_ring + (size_t)stage * P.stage_bytes;
            bulk_g2s(st, trow + e0 * tsz, tb, &full_bar[stage]);
            for (int n = 0; n + 1 < nrows; ++n)
              bulk_g2s(st + P.t_slot + n * P.q_slot, drow + ((int64_t)n * P.ld_q + e0) * qsz, qb, &full_bar[stage]);
            if (++stage == P.stages) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
  } else if (warp < kConsWarps) {
    // =============================== consumers ===============================
    const int ct = tid;  // 0..255
    int stage = 0;
    uint32_t phase = 0, j = 0;
    int jobs_done = 0;
    const float k2 = P.k2f;
    // Run every job posted so far (sampling passes over rows streamed a few us ago: L2 hits).
    auto run_jobs = [&](int upto) {
      while (jobs_done < upto) {
        const Job& jb = s_job[jobs_done % kJobSlots];
        const int jb_b = jb.b, jb_i = jb.i, kind = jb.kind;
        const Decision d = jb.d;
        const int gg = P.draft_len ? P.draft_len[jb_b] : P.k;
        const int Nd = (jb_i < gg) ? N : 0;
        const TT* trow = (const TT*)P.target + ((int64_t)jb_b * (P.k + 1) + jb_i) * P.ld_t;
        const TQ* drow = (const TQ*)P.draft + ((int64_t)jb_b * P.k + jb_i) * N * P.ld_q;
        if (jb.type == kJobSum) {
          double acc = 0.0;
#pragma unroll 2
          for (int64_t gi = cb + ct; gi < ce; gi += kConsThreads) {
            float w[8];
            group_weights<TT, TQ, kLogits, NMAX>(P, d, kind, trow, drow, Nd, gi, w);
            acc += (double)sum8(w);
          }
          acc = warp_sum(acc);
          if (lane == 0) s_scan[warp] = acc;
          cons_sync();
          if (ct == 0) {
            double zc = 0.0;
            for (int w = 0; w < kConsWarps; ++w) zc += s_scan[w];
            const int zp = (int)(jb.zcount & 1u);
            for (int r = 0; r < C; ++r) {
              cluster.map_shared_rank(&s_z[zp][0], r)[rank] = zc;
              mbar_remote_arrive(&z_bar[zp], (uint32_t)r);
            }
          }
        } else {
          const int64_t y = scan_range<TT, TQ, kLogits, NMAX, kConsThreads>(
              P, d, kind, trow, drow, Nd, cb, ce, jb.tc, jb.Z, s_scan, s_wi, &s_found, &s_margin);
          if (ct == 0) {
            SampleOut so;
            so.y = y;
            so.margin = s_margin;
            so.degenerate = jb.deg;
            so.z = (float)((kind == kWBonus) ? jb.Z * (double)d.invS : jb.Z);
            so.tx = 0.f;
            for (int n = 0; n < kMaxN; ++n) so.dx[n] = 0.f;
            *cluster.map_shared_rank(&s_y, 0) = so;
            mbar_remote_arrive(&y_bar, 0);
          }
        }
        cons_sync();  // the job slot may be reused only after everyone read it
        jobs_done++;
      }
    };
    for (int b = cid; b < P.B; b += P.ncl) {
      const int g = P.draft_len ? P.draft_len[b] : P.k;
      if (g < 1 || g > P.k) continue;
      for (int i = 0; i <= g; ++i, ++j) {
        const bool has_d = i < g;
        const int Nd = has_d ? N : 0;
        const int slot = (int)(j % kRecSlots);
        const TT* trow = (const TT*)P.target + ((int64_t)b * (P.k + 1) + i) * P.ld_t;
        const TQ* drow = (const TQ*)P.draft + ((int64_t)b * P.k + i) * N * P.ld_q;
        const int n_gath = has_d ? N * (N + 1) : 0;
        int32_t gtok = -1;
        float gval = 0.f;
        if (ct < n_gath) {  // candidate gathers, in flight during the stream
          const int n = ct % N, m = ct / N;
          gtok = P.draft_tokens[((int64_t)b * P.k + i) * N + n];
          if (gtok >= 0 && (int64_t)gtok < P.V)
            gval = (m < N) ? load_one(drow + (int64_t)m * P.ld_q, gtok) : load_one(trow, gtok);
        }
        float tmx = kNegBig, ts = 0.f, tb = -INFINITY;
        int64_t ti = -1;
        bool tbad = false, dneg = false;
        float dm[NMAX], ds[NMAX];
#pragma unroll
        for (int n = 0; n < NMAX; ++n) { dm[n] = kNegBig; ds[n] = 0.f; }
        for (int t = 0; t < ntiles; ++t) {
          mbar_wait_ring(&full_bar[stage], phase);
          const unsigned char* st = s_ring + (size_t)stage * P.stage_bytes;
          const int64_t gi = cb + (int64_t)t * kTileGroups + ct;
          if (gi < ce) {
            const bool partial = gi >= P.gfull;
            float f[8];
            smem_group<TT>(st, ct, f);
            if (partial) {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (gi * kGroup + e >= P.V) f[e] = -INFINITY;
            }
            if (greedy) {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                if (f[e] > tb) { tb = f[e]; ti = gi * kGroup + e; }
                tbad |= !(f[e] <= 3.402823466e+38f);
              }
            } else {
              const float gm = max8(f);
              if (gm > tmx) { ts *= ex2((tmx - gm) * k2); tmx = gm; }
              float e8[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) e8[e] = ex2((f[e] - tmx) * k2);
              ts += sum8(e8);
            }
#pragma unroll
            for (int n = 0; n < NMAX; ++n) {
              if (n < Nd) {
                const unsigned char* slotp = st + P.t_slot + n * P.q_slot;
                smem_group<TQ>(slotp, ct, f);
                if (partial) {
#pragma unroll
                  for (int e = 0; e < 8; ++e)
                    if (gi * kGroup + e >= P.V) f[e] = kLogits ? -INFINITY : 0.f;
                }
                if (kLogits) {
                  const float gm = max8(f);
                  if (gm > dm[n]) { ds[n] *= ex2((dm[n] - gm) * k2); dm[n] = gm; }
                  float e8[8];
#pragma unroll
                  for (int e = 0; e < 8; ++e) e8[e] = ex2((f[e] - dm[n]) * k2);
                  ds[n] += sum8(e8);
                } else {
                  // sign bits of the raw group first: the exact check only when one is set
                  const uint4 raw = reinterpret_cast<const uint4*>(slotp)[sizeof(TQ) == 2 ? ct : 2 * ct];
                  if ((raw.x | raw.y | raw.z | raw.w) & (sizeof(TQ) == 2 ? 0x80008000u : 0x80000000u) ||
                      sizeof(TQ) == 4) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) dneg |= (f[e] < 0.f);
                  }
                  ds[n] += sum8(f);
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_local(&empty_bar[stage]);
          if (++stage == P.stages) { stage = 0; phase ^= 1u; }
        }
        // ---- record slot credit: every CTA's decision warp is done with this slot's last use
        if (j >= (uint32_t)kRecSlots) {
          // record-slot credit (every CTA's decision warp is done with its last use); keep
          // serving sampling jobs while waiting, the decision warps may need them to progress
          const long long t0 = clock64();
          for (;;) {
            if (ct == 0) {
              s_final = mbar_test(&rec_free[slot], ((j / kRecSlots) - 1u) & 1u) ? 1 : 0;
              s_nready = s_posted;
              __threadfence_block();
            }
            cons_sync();
            const int ok = s_final, upto = s_nready;
            run_jobs(upto);
            cons_sync();
            if (ok) break;
            if (clock64() - t0 > (1LL << 33)) __trap();
          }
        }
        if (ct == 0) {
          s_nready = s_posted;
          __threadfence_block();
        }
        cons_sync();
        if (ct < n_gath) s_gx[slot][ct / N][ct % N] = gval;
        if (ct < Nd) s_tok[slot][ct] = gtok;
        // ---- CTA reduction -> record pushed into every CTA of the cluster ----
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
        cons_sync();
        float Mc = kNegBig;
        float dMc[NMAX];
#pragma unroll
        for (int n = 0; n < NMAX; ++n) dMc[n] = kNegBig;
        for (int w = 0; w < kConsWarps; ++w) {
          Mc = fmaxf(Mc, s_wf[w][0]);
#pragma unroll
          for (int n = 0; n < NMAX; ++n) dMc[n] = fmaxf(dMc[n], s_wf[w][1 + n]);
        }
        double tsd = 0.0;
        if (!greedy && ts != 0.f) tsd = (double)ts * exp2(((double)tmx - (double)Mc) * P.k2d);
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
        for (int n = 0; n < NMAX; ++n)
          if (n < Nd) dsd[n] = warp_sum(dsd[n]);
        const int bad = (__any_sync(0xffffffffu, tbad) ? 1 : 0) | (__any_sync(0xffffffffu, dneg) ? 2 : 0);
        if (lane == 0) {
          s_wd[warp][0] = tsd;
#pragma unroll
          for (int n = 0; n < NMAX; ++n) s_wd[warp][1 + n] = dsd[n];
          s_wbad[warp] = bad;
        }
        cons_sync();
        if (ct == 0) {
          CtaRec rec;
          rec.tmax = Mc;
          rec.targ = -1;
          rec.bad = 0;
          rec.tsum = 0.0;
          if (greedy) {
            float bv = -INFINITY;
            int64_t bi = -1;
            for (int w = 0; w < kConsWarps; ++w) {
              const float v = s_wv[w];
              const int64_t ix = s_wi[w];
              if (ix >= 0 && (bi < 0 || v > bv || (v == bv && ix < bi))) { bv = v; bi = ix; }
            }
            rec.tmax = bv;
            rec.targ = bi;
          }
          for (int w = 0; w < kConsWarps; ++w) {
            rec.tsum += s_wd[w][0];
            rec.bad |= s_wbad[w];
          }
#pragma unroll
          for (int n = 0; n < kMaxN; ++n) { rec.dmax[n] = kNegBig; rec.dsum[n] = 0.0; }
#pragma unroll
          for (int n = 0; n < NMAX; ++n) {
            rec.dmax[n] = dMc[n];
            double sacc = 0.0;
            for (int w = 0; w < kConsWarps; ++w) sacc += s_wd[w][1 + n];
            rec.dsum[n] = sacc;
          }
          for (int r = 0; r < C; ++r) {
            cluster.map_shared_rank(&s_rec[slot][0], r)[rank] = rec;
            mbar_remote_arrive(&rec_full[slot], (uint32_t)r);
          }
        }
        run_jobs(s_nready);
      }
    }
    // drain: jobs of the last positions are posted after the last record
    for (;;) {
      if (ct == 0) {
        const int fin = s_dec_done;
        __threadfence_block();
        s_nready = s_posted;
        s_final = fin;
      }
      cons_sync();
      const int upto = s_nready, fin = s_final;
      run_jobs(upto);
      if (fin && jobs_done >= upto) break;
      if (upto == jobs_done) __nanosleep(200);
    }
  } else {
    // ======================= decision warp (identical in every CTA) =======================
    uint32_t j = 0, scount = 0, ycount = 0;
    for (int b = cid; b < P.B; b += P.ncl) {
      const int g = P.draft_len ? P.draft_len[b] : P.k;
      int32_t* out = P.out_tokens + (int64_t)b * (P.k + 1);
      if (g < 1 || g > P.k) {
        if (rank == 0 && lane == 0) {
          P.accept_len[b] = -1;
          for (int jj = 0; jj <= P.k; ++jj) out[jj] = -1;
          P.status[b] = COSINE_REQ_BAD_DRAFT_LEN;
        }
        continue;
      }
      const uint64_t rid = P.rids[b];
      int first_rej = g, err = 0, sampled = 0;
      float tm = INFINITY;
      int64_t yv = -1;
      for (int i = 0; i <= g; ++i, ++j) {
        const bool has_d = i < g;
        const int Nd = has_d ? N : 0;
        const int slot = (int)(j % kRecSlots);
        if (lane == 0) {
          mbar_wait_wd(&rec_full[slot], (j / kRecSlots) & 1u);
          decide_unit<kLogits>(P, s_rec[slot], C, s_gx[slot], s_tok[slot], has_d, i, g, rid, first_rej, s_ud);
          for (int r = 0; r < C; ++r) mbar_remote_arrive(&rec_free[slot], (uint32_t)r);
          const UnitDec& u = s_ud;
          if (u.status && !err) err = u.status;
          if (!err && first_rej == g) {  // margins of the realised path: positions 0..L
            tm = fmin_(tm, u.m_fa);
            if (has_d && !u.accept) first_rej = i;
          }
          if (!err && greedy) {
            if (has_d && !u.accept && first_rej == i) yv = u.amax;
            if (!has_d && first_rej == g) yv = u.amax;
          }
          if (rank == 0) {  // per-position outputs and diagnostics
            const cosine_debug_t& D = P.dbg;
            const int64_t ou = (int64_t)b * (P.k + 1) + i;
            if (D.row_max) D.row_max[ou] = u.Mf;
            if (D.row_sumexp) D.row_sumexp[ou] = greedy ? 0.f : (float)u.S;
            if (has_d) {
              const int64_t o1 = (int64_t)b * P.k + i;
              out[i] = u.xstar;
              if (D.p_x) D.p_x[o1] = (float)u.px;
              if (D.q_x) D.q_x[o1] = (float)u.qx;
              if (D.accept_u) D.accept_u[o1] = (float)u.u;
              if (D.fused_tokens) D.fused_tokens[o1] = u.xstar;
              for (int n = 0; n < N; ++n) {
                if (D.draft_norm) D.draft_norm[o1 * N + n] = (float)u.sig[n];
                if (D.conf) D.conf[o1 * N + n] = (float)u.c[n];
                if (D.weights) D.weights[o1 * N + n] = (float)u.w[n];
              }
            }
          }
          Decision d;
          d.need = (!err && u.need && !(P.debug_flags & 1)) ? 1 : 0;
          d.kind = u.kind;
          d.xstar = u.xstar;
          d.node = u.node;
          d.u = u.u_s;
          d.k2 = P.k2f;
          d.M = u.Mf;
          d.invS = (float)(1.0 / u.S);
          for (int n = 0; n < kMaxN; ++n) {
            d.a[n] = (n < Nd) ? (float)(u.w[n] / u.sig[n]) : 0.f;
            d.dm[n] = (n < Nd) ? u.dmax[n] : 0.f;
          }
          s_dec = d;
        }
        __syncwarp();
        if (lane == 0 && s_dec.need) {
          // ---- inverse-CDF round: consumers of every CTA sum their chunk (job
          // kSum), the decision warps exchange the sums, the crossing CTA scans (job kScan) ----
          const Decision d = s_dec;
          int kind = d.kind, deg = 0;
          for (;;) {
            const int zp = (int)(scount & 1u);
            Job jb;
            jb.type = kJobSum; jb.b = b; jb.i = i; jb.kind = kind; jb.deg = deg; jb.zcount = scount;
            jb.tc = 0.0; jb.Z = 0.0; jb.d = d;
            s_job[s_posted % kJobSlots] = jb;
            __threadfence_block();
            s_posted = s_posted + 1;
            mbar_wait_wd(&z_bar[zp], (scount >> 1) & 1u);
            scount++;
            double Z = 0.0;
            for (int c = 0; c < C; ++c) Z += s_z[zp][c];
            if (!(Z > 0.0) && (kind == kWResidual || kind == kWPoint)) {
              kind = kWProb;  // all mass cancelled: resample from o (reading #11)
              deg = 1;
              continue;
            }
            int cstar = -1;
            double tc = 0.0;
            if (Z > 0.0) {
              const double t = d.u * Z;
              double O = 0.0;
              for (int c = 0; c < C; ++c) {
                const double zz = s_z[zp][c];
                if (O + zz > t) { cstar = c; tc = t - O; break; }
                O += zz;
              }
            }
            if (rank == cstar) {
              jb.type = kJobScan; jb.kind = kind; jb.deg = deg; jb.tc = tc; jb.Z = Z;
              s_job[s_posted % kJobSlots] = jb;
              __threadfence_block();
              s_posted = s_posted + 1;
            }
            sampled = (cstar >= 0) ? 1 : -1;
            break;
          }
        }
        __syncwarp();
      }
      // ---------------- request outputs (CTA 0) ----------------
      if (rank == 0 && lane == 0) {
        float zmass = NAN;
        int degenerate = 0;
        if (sampled == 1) {  // always consumed: keeps y_bar's phase in step
          mbar_wait_wd(&y_bar, ycount & 1u);
          ycount++;
        }
        if (err) {
          P.accept_len[b] = -1;
          for (int jj = 0; jj <= P.k; ++jj) out[jj] = -1;
          P.status[b] = err;
        } else {
          const int L = first_rej;
          int flags = 0;
          if (!greedy) {
            if (sampled == 1) {
              yv = s_y.y;
              tm = fmin_(tm, s_y.margin);
              degenerate = s_y.degenerate;
              zmass = s_y.z;
            } else {
              yv = -1;
              flags |= 0xff;
            }
          }
          out[L] = (int32_t)yv;
          for (int jj = L + 1; jj <= P.k; ++jj) out[jj] = -1;
          P.accept_len[b] = L;
          flags |= (degenerate ? COSINE_INFO_DEGENERATE_RESIDUAL : 0) | (tm < 1e-6f ? COSINE_INFO_NEAR_TIE : 0);
          P.status[b] = flags;
          if (P.dbg.residual_mass) P.dbg.residual_mass[b] = zmass;
          if (P.dbg.tie_margin) P.dbg.tie_margin[b] = tm;
        }
      }
      __syncwarp();
    }
    if (lane == 0) {
      __threadfence_block();
      s_dec_done = 1;
    }
  }
  cluster.sync();  // no CTA leaves while a peer may still write into its shared memory
}

}  // namespace cosine
