// cosine_abi.cu — host side of libcosine_verify.so: the C ABI (include/cosine_verify.h),
// argument checks, context / scratch ownership, launch configuration, NCCL for the
// vocabulary-sharded mode, and the kernels that do not depend on the row dtypes.
//
// Kernels (all hand-written for sm_100a; nothing on this path is a contraction, so no tensor
// cores — it is HBM-bound):
//   cosine_verify_batch (1 GPU, ARGMAX)   stats -> decide -> resample (PDL, device counters)
//   cosine_verify_batch (vocab-sharded)   stats -> pack -> all-gather -> decide -> resample ->
//                                         all-gather -> sample -> all-gather -> finish
//   cosine_verify_batch_lazy (NEXT-1)     rounds of stats + lazy_decide, then resample
//   cosine_verify_tree[_lazy] (A10)       stats + tree_decide + tree_walk (cosine_tree.cuh)
//   cosine_fuse_step / route_update / tree_select (NEXT-2..4)
// See DESIGN.md §5 for the roofline, byte accounting and the B200 design choices.

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

#include "cosine_dispatch.h"
#include "cosine_fuse_step.cuh"
#include "cosine_route.cuh"
#include "cosine_shard.cuh"
#include "cosine_tree_select.cuh"
#include "cosine_verify.h"

namespace cosine {

__global__ void __launch_bounds__(kThreads) fuse_finish_kernel(const SplitParams P) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the decisions (PDL)
  const int b = blockIdx.x * kThreads + threadIdx.x;
  if (b >= P.B) return;
  int err = 0;
  float tm = INFINITY;
  for (int i = 0; i < P.k && !err; ++i) {
    const PosDec& pd = P.pdec[(int64_t)b * P.k + i];
    err = pd.status;
    tm = fmin_(tm, pd.m_fa);
  }
  if (err)
    for (int i = 0; i < P.k; ++i) P.fuse_tokens[(int64_t)b * P.k + i] = -1;
  P.status[b] = err ? err : (tm < 1e-6f ? COSINE_INFO_NEAR_TIE : 0);
}

void kernel_set(cosine_dtype_t tt, cosine_dtype_t tq, bool logits, int N, KernelSet* ks) {
  if (tt == COSINE_BF16 && tq == COSINE_BF16) kernel_set_bb(logits, N, ks);
  else if (tt == COSINE_BF16 && tq == COSINE_F32) kernel_set_bf(logits, N, ks);
  else if (tt == COSINE_F32 && tq == COSINE_BF16) kernel_set_fb(logits, N, ks);
  else kernel_set_ff(logits, N, ks);
}

}  // namespace cosine

// =====================================================================================
// C ABI
// =====================================================================================
using namespace cosine;

struct cosine_ctx_s {
  cosine_config_t cfg;
  int64_t V;
  PartRec* parts = nullptr;
  PosDec* pdec = nullptr;
  int32_t* counters = nullptr;
  size_t counters_bytes = 0;
  NodeDec* ndec = nullptr;
  ChildPQ* cpq = nullptr;
  double* segsum = nullptr;
  size_t segsum_cap = 0;
  int tiny_cap[2] = {-1, -1};  // co-resident tiny_kernel CTAs (NMAX 4 / 8), -1 = not queried
  float* slices = nullptr;  // SAMPLE selection: 64-group slice sums of the drafter rows
  size_t slices_cap = 0;    // floats
  // optional live timing of the dominant kernel (stats_kernel) with CUDA events on the stream
  int prof_on = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev;
  size_t prof_n = 0;
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
  bool vgroup = false;  // a cosine_verify_init_vgroup context (device copies instead of NCCL)
  // in-kernel exchange over NVLink peer memory: this rank's gather block [rec_all | zall | yall |
  // arrival counters] (one allocation, shared with the peers through CUDA IPC) and the peers'
  // blocks mapped into this process; p2p = false -> the NCCL all-gathers
  bool p2p = false;
  char* xblock = nullptr;
  size_t xrec = 0, xz = 0, xy = 0;  // byte offsets of zall, yall and the counters in a block
  char* peer_block[kMaxPeers] = {};
  unsigned long long arrivals[3] = {0, 0, 0};  // cumulative arrival targets (same on every rank)
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

// Chunk CTAs per unit of the streaming kernels: ~8 groups (64 elements per row) per thread,
// then widen while the grid has fewer than ~8 CTAs per SM.
int stats_chunks(const cosine_ctx_t ctx, int64_t units, int64_t ngroups, int per_thread = 8) {
  if (ctx->cfg.cluster_size > 0) return ctx->cfg.cluster_size;
  int C = 1;
  while (C < kMaxC && ngroups > (int64_t)C * kThreads * per_thread) C *= 2;
  while (C < kMaxC && units * C < 148 * 8 && ngroups >= (int64_t)C * 2 * kThreads) C *= 2;
  return C;
}

void fill_scratch(const cosine_ctx_t ctx, SplitParams& S, int C) {
  S.C = C;
  S.cg = (S.ngroups + C - 1) / C;
  S.nseg = (S.ngroups + kTileGroups - 1) / kTileGroups;
  // tiles per resample CTA: 8 for large batches; fewer (more, shorter CTAs) while the final
  // draws of the batch fill less than ~2 waves — small batches are latency-bound
  S.tpc = kSegTilesPerCta;  // (8 / 12 / 16 measured equal on c3 and c5)
  while (S.tpc > 1 && (int64_t)S.B * ((S.nseg + S.tpc - 1) / S.tpc) < 2 * 148 * 5) S.tpc /= 2;
  S.spr = (int)((S.nseg + S.tpc - 1) / S.tpc);
  S.parts = ctx->parts;
  S.pdec = ctx->pdec;
  S.segsum = ctx->segsum;
  S.counters = ctx->counters;
  S.dcnt = ctx->counters + std::max(ctx->cfg.max_batch, 1);
  S.ucnt = ctx->counters + 2 * (size_t)std::max(ctx->cfg.max_batch, 1);
  S.b_off = 0;
  S.nb = S.B;
}

// Optional live timing of the dominant kernel with CUDA events on its stream.
std::pair<cudaEvent_t, cudaEvent_t> prof_events(cosine_ctx_t ctx) {
  if (!ctx->prof_on) return {nullptr, nullptr};
  if (ctx->prof_n == ctx->prof_ev.size()) {
    cudaEvent_t a0, a1;
    cudaEventCreate(&a0);
    cudaEventCreate(&a1);
    ctx->prof_ev.emplace_back(a0, a1);
  }
  return ctx->prof_ev[ctx->prof_n++];
}

// The split path: stats_kernel -> decide_kernel -> resample_kernel, the latter two programmatic
// dependents waiting per unit / per request on device counters (scheduled into the previous
// grid's tail wave; the waits always end because every CTA they wait for is resident or done).
#ifdef COSINE_TRACE
// instrumentation build: one device buffer of phase timestamps, read by cosine_trace_read
static unsigned long long* g_trace = nullptr;
static size_t g_trace_n = 0;
unsigned long long* cosine_trace_buffer(size_t n) {
  if (n > g_trace_n) {
    cudaFree(g_trace);
    cudaMalloc(&g_trace, n * sizeof(unsigned long long));
    g_trace_n = n;
  }
  cudaMemset(g_trace, 0, g_trace_n * sizeof(unsigned long long));
  return g_trace;
}
size_t cosine_trace_copy(unsigned long long* host, size_t n) {
  cudaDeviceSynchronize();
  n = std::min(n, g_trace_n);
  if (n) cudaMemcpy(host, g_trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return n;
}
#endif

// Small batches (ARGMAX): the whole call as one cooperative launch of tiny_kernel when its
// (unit, chunk) grid is co-resident and the request's CTAs cover its final draw's tiles.
// Returns false (nothing enqueued) when the batch does not qualify.
bool launch_tiny(cosine_ctx_t ctx, cudaStream_t stream, SplitParams& S, const KernelSet& ks, cosine_status_t* st) {
  const int64_t units = (int64_t)S.B * (S.k + 1);
  const int slot = S.N <= 4 ? 0 : 1;
  if (ctx->tiny_cap[slot] < 0) {
    int occ = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ks.tiny, kThreads, 0) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->cfg.device) != cudaSuccess) {
      cudaGetLastError();
      occ = 0;
    }
    ctx->tiny_cap[slot] = occ * sms;
  }
  const int64_t cap = ctx->tiny_cap[slot];
  if (ctx->cfg.cluster_size > 0 || units > cap) return false;
  int C = stats_chunks(ctx, units, S.ngroups);
  while (C < kMaxC && units * 2 * C <= cap && S.ngroups >= (int64_t)C * kThreads) C *= 2;
  while (C > 1 && units * C > cap) C /= 2;
  fill_scratch(ctx, S, C);
  const int64_t per_req = (int64_t)(S.k + 1) * C;
  S.tpc = (int)((S.nseg + per_req - 1) / per_req);
  if (S.tpc > kSegTilesPerCta) return false;
  S.spr = (int)((S.nseg + S.tpc - 1) / S.tpc);
  if ((size_t)S.B * (size_t)S.nseg > ctx->segsum_cap) return false;
  S.fused = 1;
#ifdef COSINE_TRACE
  S.trace = cosine_trace_buffer((size_t)units * C * 16);
#endif
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.gridDim = dim3((unsigned)(units * C), 1, 1);
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // co-residency: the parts wait on other CTAs
  at[0].val.cooperative = 1;
  lc.attrs = at;
#ifdef COSINE_TRACE_NONCOOP  // (latency study only)
  lc.numAttrs = 0;
#else
  lc.numAttrs = 1;
#endif
  const auto pe = prof_events(ctx);
  if (pe.first) cudaEventRecord(pe.first, stream);
  const cudaError_t e = cudaLaunchKernelEx(&lc, ks.tiny, S);
  if (pe.second) cudaEventRecord(pe.second, stream);
  if (e == cudaErrorCooperativeLaunchTooLarge) {  // (not expected: the grid fits the query)
    cudaGetLastError();
    return false;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    *st = fail(ctx, COSINE_ERR_CUDA, std::string("verify kernel (one launch): ") + cudaGetErrorString(e));
    return true;
  }
  ctx->last_launches = 1;
  ctx->last_cluster = C;
  *st = COSINE_OK;
  return true;
}

cosine_status_t launch_split3(cosine_ctx_t ctx, cudaStream_t stream, SplitParams& S, const KernelSet& ks,
                              bool sample) {
  const int64_t units = (int64_t)S.B * (S.k + 1);
  if (!sample && !S.lazy && !S.tree && S.mode == kSplitVerify && ks.tiny) {
    cosine_status_t st = COSINE_OK;
    if (launch_tiny(ctx, stream, S, ks, &st)) return st;
  }
  fill_scratch(ctx, S, stats_chunks(ctx, units, S.ngroups));
  if ((size_t)S.B * (size_t)S.nseg > ctx->segsum_cap)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "segment scratch too small");
  S.fused = 1;
  // SAMPLE over probability drafts: the statistics pass keeps 64-group slice sums and the draw
  // runs a warp per unit (sample_decide_w_kernel); otherwise a CTA per unit scans the chunk
  S.nsl = (S.cg + kSliceGroups - 1) / kSliceGroups;
  const bool sliced = sample && !S.greedy && ks.stats_slices && ctx->slices && !S.lazy && !S.tree &&
                      (size_t)units * S.C * S.nsl * S.N <= ctx->slices_cap;
  S.slices = sliced ? ctx->slices : nullptr;
  const bool warp_b1 = !sample || sliced;
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  const auto pe = prof_events(ctx);
#ifdef COSINE_TRACE  // [stats grid | decide grid | resample grid] x 16 slots
  const size_t n_st = (size_t)units * S.C, n_de = (size_t)units, n_rs = (size_t)S.B * S.spr;
  unsigned long long* tb = cosine_trace_buffer(16 + (n_st + n_de + n_rs) * 16);
  const unsigned long long hdr[3] = {n_st, n_de, n_rs};  // header: the three grids' sizes
  cudaMemcpy(tb, hdr, sizeof(hdr), cudaMemcpyHostToDevice);
  tb += 16;
  S.trace = tb;
#endif
  if (pe.first) cudaEventRecord(pe.first, stream);
  lc.gridDim = dim3((unsigned)(units * S.C), 1, 1);
  cudaError_t e = cudaLaunchKernelEx(&lc, sliced ? ks.stats_slices : ks.stats, S);
#ifdef COSINE_TRACE
  S.trace = tb + n_st * 16;
#endif
  if (pe.second) cudaEventRecord(pe.second, stream);
  if (e == cudaSuccess) {
    // ARGMAX and sliced SAMPLE: a warp per unit; SAMPLE otherwise: a CTA per unit (the draw
    // scans one chunk block-wide)
    lc.gridDim = dim3((unsigned)(warp_b1 ? (units + kWarps - 1) / kWarps : units), 1, 1);
    lc.attrs = pe.second ? nullptr : at;  // (an event record between the two breaks PDL)
    lc.numAttrs = pe.second ? 0 : 1;
    e = cudaLaunchKernelEx(&lc, !sample ? ks.decide : (sliced ? ks.sample_decide_w : ks.sample_decide), S);
  }
  if (e == cudaSuccess) {
#ifdef COSINE_TRACE
    S.trace = tb + (n_st + n_de) * 16;
#endif
    lc.gridDim = dim3((unsigned)(S.B * S.spr), 1, 1);
    lc.attrs = at;
    lc.numAttrs = 1;
    e = cudaLaunchKernelEx(&lc, ks.resample, S);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    // a later launch failed after stats_kernel was enqueued: its per-unit counts must not leak
    // into the next call (the dependents reset them); clear the counter block on the stream
    cudaMemsetAsync(ctx->counters, 0, ctx->counters_bytes, stream);
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("verify kernels: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = 3;
  ctx->last_cluster = S.C;
  return COSINE_OK;
}

// cosine_verify_batch on one GPU.
cosine_status_t launch_split(cosine_ctx_t ctx, cudaStream_t stream, SplitParams& S,
                             cosine_dtype_t tt, cosine_dtype_t tq, bool logits, bool sample) {
  KernelSet ks;
  memset(&ks, 0, sizeof(ks));
  kernel_set(tt, tq, logits, S.N, &ks);
  return launch_split3(ctx, stream, S, ks, sample);
}

// ---------------------------------------------------------------------------------------
// Vocabulary-sharded verification (cosine_shard.cuh): four phases with three exchanges:
//   A: stats_kernel (local columns) -> shard_pack_kernel      X1: records   [G][units][words]
//   B: shard_decide_kernel -> resample_kernel (local masses)  X2: masses    [G][B] doubles
//   C: shard_sample_kernel (the owner of t scans)             X3: tokens    [G][B] YRec
//   D: shard_finish_kernel (replicated outputs)
// ---------------------------------------------------------------------------------------
void shard_setup(cosine_ctx_t ctx, SplitParams& S) {
  const int64_t units = (int64_t)S.B * (S.k + 1);
  fill_scratch(ctx, S, stats_chunks(ctx, units, S.ngroups));
  S.fused = 0;
  S.ucount = 1;  // shard_pack_kernel waits per unit (scheduled into the statistics' tail)
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
}

struct ShardLaunch {
  cudaLaunchConfig_t lc;
  cudaLaunchAttribute at[1];
  explicit ShardLaunch(cudaStream_t s) {
    memset(&lc, 0, sizeof(lc));
    lc.blockDim = dim3(kThreads, 1, 1);
    lc.stream = s;
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
  }
  cudaError_t operator()(SplitFn f, unsigned grid, bool pdl, const SplitParams& S) {
    lc.gridDim = dim3(grid, 1, 1);
    lc.attrs = pdl ? at : nullptr;
    lc.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&lc, f, S);
  }
};

// Phase A of a slice: local statistics and the slice's records.
cudaError_t shard_phase_a(cosine_ctx_t ctx, cudaStream_t s, const SplitParams& S, const KernelSet& ks,
                          const char** stage) {
  ShardLaunch L(s);
  const int64_t units = (int64_t)S.B * (S.k + 1);
  *stage = "stats";
  const auto pe = prof_events(ctx);
  if (pe.first) cudaEventRecord(pe.first, s);
  cudaError_t e = L(ks.stats, (unsigned)(units * S.C), false, S);
  if (pe.second) cudaEventRecord(pe.second, s);
  if (e == cudaSuccess) {
    *stage = "pack";
    e = L(ks.shard_pack, (unsigned)((units + kWarps - 1) / kWarps), pe.second == nullptr, S);
  }
  return e;
}
// Phase B: decisions from the gathered records, local masses of the final draw.
cudaError_t shard_phase_b(cudaStream_t s, const SplitParams& S, const KernelSet& ks, bool logits, const char** stage) {
  // p2p: the consumers wait on the arrival counters (their own rank's producer arrives too), so
  // they are launched as programmatic dependents: their launch latency hides under the producer
  ShardLaunch L(s);
  const int64_t units = (int64_t)S.B * (S.k + 1);
  *stage = "decide";
  cudaError_t e = L(logits ? shard_decide_kernel<true> : shard_decide_kernel<false>,
                    (unsigned)((units + kWarps - 1) / kWarps), S.p2p != 0, S);
  if (e == cudaSuccess) {
    *stage = "resample";
    e = L(ks.resample, (unsigned)(S.B * S.spr), true, S);
  }
  return e;
}
cudaError_t shard_phase_c(cudaStream_t s, const SplitParams& S, const KernelSet& ks, const char** stage) {
  ShardLaunch L(s);
  *stage = "sample";
  return L(ks.shard_sample, (unsigned)S.B, S.p2p != 0, S);
}
cudaError_t shard_phase_d(cudaStream_t s, const SplitParams& S, const char** stage) {
  ShardLaunch L(s);
  *stage = "finish";
  return L(shard_finish_kernel, (unsigned)((S.B + kWarps - 1) / kWarps), S.p2p != 0, S);
}
size_t shard_x_bytes(const SplitParams& S, int x) {  // bytes one rank contributes to exchange x
  if (x == 1) return (size_t)S.B * (S.k + 1) * S.rec_words * 4;
  if (x == 2) return (size_t)S.B * sizeof(double);
  return (size_t)S.B * sizeof(YRec);
}
ncclResult_t shard_allgather(cosine_ctx_t ctx, cudaStream_t s, const SplitParams& S, int x) {
  const void* src = x == 1 ? (const void*)S.rec_send : (x == 2 ? (const void*)S.zsend : (const void*)S.ysend);
  void* dst = x == 1 ? (void*)S.rec_all : (x == 2 ? (void*)S.zall : (void*)S.yall);
  return ncclAllGather(src, dst, shard_x_bytes(S, x), ncclUint8, ctx->comm, s);
}

cosine_status_t shard_fail(cosine_ctx_t ctx, cudaStream_t s, cudaError_t e, ncclResult_t r, const char* stage) {
  cudaGetLastError();
  cudaMemsetAsync(ctx->counters, 0, ctx->counters_bytes, s);  // (as in launch_split3)
  cudaGetLastError();
  ctx->last_launches = 0;
  if (e != cudaSuccess)
    return fail(ctx, COSINE_ERR_CUDA, std::string("sharded verify (") + stage + "): " + cudaGetErrorString(e));
  return fail(ctx, COSINE_ERR_NCCL, std::string("sharded verify all-gather: ") + ncclGetErrorString(r));
}

// Collective (init): share this rank's gather block with the other ranks through CUDA IPC (the
// handles travel by one NCCL all-gather) and map theirs.  Any failure leaves p2p off: the call
// then uses the NCCL all-gathers.
void p2p_attach(cosine_ctx_t ctx) {
  const int G = ctx->cfg.nranks, rank = ctx->cfg.rank;
  cudaIpcMemHandle_t mine;
  bool ok = cudaIpcGetMemHandle(&mine, ctx->xblock) == cudaSuccess;
  void* dev = nullptr;
  std::vector<cudaIpcMemHandle_t> all(G);
  cudaStream_t s = nullptr;
  ok = ok && cudaMalloc(&dev, sizeof(cudaIpcMemHandle_t) * (G + 1)) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess;
  // every rank takes part in the all-gather (a rank whose handle failed sends zeros)
  if (dev) {
    cudaMemcpy((char*)dev + sizeof(mine) * G, &mine, sizeof(mine), cudaMemcpyHostToDevice);
    const ncclResult_t r = ncclAllGather((char*)dev + sizeof(mine) * G, dev, sizeof(mine), ncclUint8, ctx->comm, s);
    ok = ok && r == ncclSuccess && cudaStreamSynchronize(s) == cudaSuccess;
    ok = ok && cudaMemcpy(all.data(), dev, sizeof(mine) * G, cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  for (int g = 0; g < G && ok; ++g) {
    if (g == rank) {
      ctx->peer_block[g] = ctx->xblock;
      continue;
    }
    void* p = nullptr;
    ok = cudaIpcOpenMemHandle(&p, all[g], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    ctx->peer_block[g] = (char*)p;
  }
  // every rank must agree: p2p only if it is on everywhere
  int flag = ok ? 1 : 0;
  if (dev) {
    cudaMemcpy(dev, &flag, sizeof(int), cudaMemcpyHostToDevice);
    if (ncclAllReduce(dev, dev, 1, ncclInt32, ncclMin, ctx->comm, s) == ncclSuccess && cudaStreamSynchronize(s) == cudaSuccess)
      cudaMemcpy(&flag, dev, sizeof(int), cudaMemcpyDeviceToHost);
    else
      flag = 0;
  }
  if (s) cudaStreamDestroy(s);
  if (dev) cudaFree(dev);
  cudaGetLastError();
  ctx->p2p = flag != 0;
  if (!ctx->p2p)
    for (int g = 0; g < G; ++g) {
      if (ctx->peer_block[g] && ctx->peer_block[g] != ctx->xblock) cudaIpcCloseMemHandle(ctx->peer_block[g]);
      ctx->peer_block[g] = nullptr;
    }
}

// The peer pointers and arrival targets of one sharded call (p2p): rank r's records go to
// [r][units][words] of every peer's block, its masses to [r][B], its tokens to [r][B].
void p2p_params(cosine_ctx_t ctx, SplitParams& S) {
  S.p2p = 1;
  const int G = S.G, r = S.rank;
  const int64_t units = (int64_t)S.B * (S.k + 1);
  for (int g = 0; g < G; ++g) {
    char* blk = ctx->peer_block[g];
    S.rec_peer[g] = (uint32_t*)blk + (int64_t)r * units * S.rec_words;
    S.z_peer[g] = (double*)(blk + ctx->xz) + (int64_t)r * S.B;
    S.y_peer[g] = (YRec*)(blk + ctx->xy) + (int64_t)r * S.B;
    S.cnt_peer[g] = (unsigned long long*)(blk + ctx->xrec);
  }
  S.cnt_own = (unsigned long long*)(ctx->xblock + ctx->xrec);
  const unsigned long long pack_ctas = (unsigned long long)((units + kWarps - 1) / kWarps);
  ctx->arrivals[0] += (unsigned long long)G * pack_ctas;
  ctx->arrivals[1] += (unsigned long long)G * (unsigned long long)S.B;
  ctx->arrivals[2] += (unsigned long long)G * (unsigned long long)S.B;
  for (int x = 0; x < 3; ++x) S.tgt[x] = ctx->arrivals[x];
}

// One rank's collective call (NCCL): the four phases on `stream` with an all-gather after each
// of the first three.  (Request slices whose exchanges ran on a second stream under the next
// slice's statistics were measured slower on 2 B200s: 1 / 2 / 4 / 8 slices -> 1024 / 1046 / 1097 /
// 1288 us per c5 call — the slices' B phases take SMs and bandwidth from the statistics stream;
// profiles/r2_c5_slices.md.)
cosine_status_t launch_shard(cosine_ctx_t ctx, cudaStream_t stream, SplitParams& F, cosine_dtype_t tt,
                             cosine_dtype_t tq, bool logits) {
  KernelSet ks;
  kernel_set(tt, tq, logits, F.N, &ks);
  shard_setup(ctx, F);
  if ((size_t)F.B * (size_t)F.nseg > ctx->segsum_cap)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "segment scratch too small");
  const char* stage = "stats";
  ncclResult_t r = ncclSuccess;
  if (ctx->p2p) p2p_params(ctx, F);  // in-kernel exchange: no all-gathers
  cudaError_t e = shard_phase_a(ctx, stream, F, ks, &stage);
  if (e == cudaSuccess && !F.p2p) r = shard_allgather(ctx, stream, F, 1);
  if (e == cudaSuccess && r == ncclSuccess) e = shard_phase_b(stream, F, ks, logits, &stage);
  if (e == cudaSuccess && r == ncclSuccess && !F.p2p) r = shard_allgather(ctx, stream, F, 2);
  if (e == cudaSuccess && r == ncclSuccess) e = shard_phase_c(stream, F, ks, &stage);
  if (e == cudaSuccess && r == ncclSuccess && !F.p2p) r = shard_allgather(ctx, stream, F, 3);
  if (e == cudaSuccess && r == ncclSuccess) e = shard_phase_d(stream, F, &stage);
  if (e != cudaSuccess || r != ncclSuccess) return shard_fail(ctx, stream, e, r, stage);
  ctx->last_launches = 6;
  ctx->last_cluster = F.C;
  return COSINE_OK;
}

// The call of a virtual group (cosine_verify_batch_vgroup): G contexts, one stream, phase by
// phase over all ranks, each exchange done by device copies into every rank's gather buffer in
// rank order — the same kernels, slices and record layouts as launch_shard.
cosine_status_t launch_shard_vgroup(const cosine_ctx_t* ctxs, int G, cudaStream_t stream, SplitParams* F,
                                    cosine_dtype_t tt, cosine_dtype_t tq, bool logits, bool p2p) {
  KernelSet ks;
  kernel_set(tt, tq, logits, F[0].N, &ks);
  for (int g = 0; g < G; ++g) {
    shard_setup(ctxs[g], F[g]);
    if ((size_t)F[g].B * (size_t)F[g].nseg > ctxs[g]->segsum_cap)
      return fail(ctxs[g], COSINE_ERR_INVALID_ARGUMENT, "segment scratch too small");
  }
  const char* stage = "stats";
  cudaError_t e = cudaSuccess;
  if (p2p) {  // the in-kernel exchange, peers = the other contexts' blocks on this device
    for (int g = 0; g < G; ++g) {
      for (int h = 0; h < G; ++h) ctxs[g]->peer_block[h] = ctxs[h]->xblock;
      p2p_params(ctxs[g], F[g]);
    }
  }
  auto exchange = [&](int x) {
    if (p2p) return;
    for (int g = 0; g < G && e == cudaSuccess; ++g) {
      const size_t n = shard_x_bytes(F[g], x);
      const void* src = x == 1 ? (const void*)F[g].rec_send
                               : (x == 2 ? (const void*)F[g].zsend : (const void*)F[g].ysend);
      for (int h = 0; h < G && e == cudaSuccess; ++h) {
        char* dst = (char*)(x == 1 ? (void*)F[h].rec_all : (x == 2 ? (void*)F[h].zall : (void*)F[h].yall));
        e = cudaMemcpyAsync(dst + (size_t)g * n, src, n, cudaMemcpyDeviceToDevice, stream);
      }
    }
  };
  for (int g = 0; g < G && e == cudaSuccess; ++g) e = shard_phase_a(ctxs[g], stream, F[g], ks, &stage);
  exchange(1);
  for (int g = 0; g < G && e == cudaSuccess; ++g) e = shard_phase_b(stream, F[g], ks, logits, &stage);
  exchange(2);
  for (int g = 0; g < G && e == cudaSuccess; ++g) e = shard_phase_c(stream, F[g], ks, &stage);
  exchange(3);
  for (int g = 0; g < G && e == cudaSuccess; ++g) e = shard_phase_d(stream, F[g], &stage);
  if (e != cudaSuccess) return shard_fail(ctxs[0], stream, e, ncclSuccess, stage);
  for (int g = 0; g < G; ++g) ctxs[g]->last_launches = 6;
  return COSINE_OK;
}

// Lazy verification (NEXT-1): rounds r = 0..k of (stats of position r of the requests still
// verifying -> their decisions), then the final draws.  2 (k + 1) + 1 launches on `stream`.
cosine_status_t launch_lazy(cosine_ctx_t ctx, cudaStream_t stream, SplitParams& S, cosine_dtype_t tt,
                            cosine_dtype_t tq, bool logits) {
  KernelSet ks;
  kernel_set(tt, tq, logits, S.N, &ks);
  const int C = stats_chunks(ctx, S.B, S.ngroups);
  fill_scratch(ctx, S, C);
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
  // rounds of kLazySpan positions (measured on c3: 1 -> 393 us, 2 -> 366 us, 3 -> 372 us); each
  // round's decide kernel is scheduled into the stats tail (PDL) and waits per position
  S.lazy_span = kLazySpan;
  S.fused = 1;
  for (int r = 0; r <= S.k && e == cudaSuccess; r += S.lazy_span) {
    S.lazy = r + 1;
    lc.gridDim = dim3((unsigned)((int64_t)S.B * S.lazy_span * S.C), 1, 1);
    lc.attrs = nullptr;  // stream order: the round reads the previous round's lz
    lc.numAttrs = 0;
    e = cudaLaunchKernelEx(&lc, ks.stats, S);
    if (e == cudaSuccess) {
      lc.gridDim = dim3((unsigned)((S.B + kWarps - 1) / kWarps), 1, 1);
      lc.attrs = at;
      lc.numAttrs = 1;
      e = cudaLaunchKernelEx(&lc, ks.lazy_decide, S);
    }
    launches += 2;
  }
  S.lazy = 0;
  S.fused = 0;  // the final draws wait for the last round's grid (griddepcontrol.wait)
  if (e == cudaSuccess) {
    lc.gridDim = dim3((unsigned)(S.B * S.spr), 1, 1);
    lc.attrs = at;
    lc.numAttrs = 1;
    e = cudaLaunchKernelEx(&lc, ks.resample, S);
    launches += 1;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaMemsetAsync(ctx->counters, 0, ctx->counters_bytes, stream);  // (as in launch_split3)
    cudaMemsetAsync(ctx->lz, 0, (size_t)std::max(ctx->cfg.max_batch, 1) * sizeof(int32_t), stream);
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("lazy verify kernels: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = launches;
  ctx->last_cluster = C;
  return COSINE_OK;
}

// The vocabulary geometry and temperature constants of a call.
struct CallDims {
  int64_t V, ngroups, gfull;
  int greedy;
  float k2f;  // log2(e) / T (T = 0: greedy, 0)
  double k2d;
  uint64_t seed;
};
CallDims call_dims(const cosine_ctx_t ctx, float T) {
  CallDims D;
  D.V = ctx->V;
  D.ngroups = (ctx->V + kGroup - 1) / kGroup;
  D.gfull = ctx->V / kGroup;
  D.greedy = (T == 0.f);
  D.k2d = (T > 0.f) ? 1.4426950408889634 / (double)T : 0.0;
  D.k2f = (float)D.k2d;
  D.seed = ctx->cfg.seed;
  return D;
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

static cosine_status_t init_impl(const cosine_config_t* cfg, cosine_ctx_t* out, bool vgroup) {
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
  if (cfg->nranks > 1 && !cfg->nccl_unique_id && !vgroup)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "nranks > 1 needs nccl_unique_id (cosine_nccl_unique_id on rank 0)");
  if (cfg->exchange != 0 && cfg->exchange != 1)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "exchange must be 0 (automatic) or 1 (NCCL)");
  if (cfg->cluster_size != 0 && cfg->cluster_size != 1 && cfg->cluster_size != 2 &&
      cfg->cluster_size != 4 && cfg->cluster_size != 8 && cfg->cluster_size != 16)
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "cluster_size must be 0, 1, 2, 4, 8 or 16");
  cosine_ctx_t ctx = new (std::nothrow) cosine_ctx_s();
  if (!ctx) return fail(nullptr, COSINE_ERR_OUT_OF_MEMORY, "host allocation failed");
  ctx->cfg = *cfg;
  ctx->vgroup = vgroup;
  ctx->cfg.nccl_unique_id = nullptr;
  ctx->V = cfg->vocab_end - cfg->vocab_begin;
  DeviceGuard dg(cfg->device);
  const size_t nb = (size_t)std::max(cfg->max_batch, 1);
  cudaError_t e = cudaSuccess;
  const size_t nu = nb * (size_t)std::max(cfg->max_draft_len + 1, std::max(cfg->max_tree_nodes, 1));
  const size_t nt = nb * (size_t)std::max(cfg->max_tree_nodes, 1);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->ndec, nt * sizeof(NodeDec));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->cpq, nt * sizeof(ChildPQ));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->parts, nu * kMaxC * sizeof(PartRec));
  ctx->parts_cap = nu * kMaxC;
  if (e == cudaSuccess) e = cudaMalloc(&ctx->pdec, nu * sizeof(PosDec));
  // counters: [B] kernel-B CTAs per request | [B] decided units per request | [B][k+1] chunks per unit
  const size_t ncnt = 2 * nb + nb * (size_t)(cfg->max_draft_len + 1);
  ctx->counters_bytes = ncnt * sizeof(int32_t);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->counters, ncnt * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->lz, nb * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemset(ctx->counters, 0, ncnt * sizeof(int32_t));
  ctx->segsum_cap = nb * (size_t)((ctx->V + (int64_t)kTileElems - 1) / kTileElems);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->segsum, ctx->segsum_cap * sizeof(double));
  if (e == cudaSuccess && cfg->nranks == 1 && cfg->draft_kind == COSINE_DRAFT_PROBS) {
    // slice sums for SAMPLE selection: per unit and drafter <= ceil(groups / kSliceGroups) +
    // kMaxC floats (chunks round up), i.e. ~1/256 of a bf16 drafter row
    const size_t units = nb * (size_t)(cfg->max_draft_len + 1);
    const size_t per = (size_t)((ctx->V + kGroup * kSliceGroups - 1) / (kGroup * kSliceGroups)) + kMaxC;
    ctx->slices_cap = units * per * (size_t)cfg->max_drafters;
    e = cudaMalloc(&ctx->slices, ctx->slices_cap * sizeof(float));
  }
  if (e == cudaSuccess && cfg->nranks > 1) {  // vocabulary-sharded: exchange buffers + communicator
    const size_t units = nb * (size_t)(cfg->max_draft_len + 1);
    const size_t rb = units * (size_t)shard_rec_words(cfg->max_drafters) * 4;
    const size_t G = (size_t)cfg->nranks;
    e = cudaMalloc(&ctx->rec_send, rb);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->zsend, nb * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&ctx->ysend, nb * sizeof(YRec));
    // the gather buffers and the arrival counters in one block (the unit of IPC sharing)
    ctx->xz = (rb * G + 255) / 256 * 256;
    ctx->xy = ctx->xz + (nb * sizeof(double) * G + 255) / 256 * 256;
    ctx->xrec = ctx->xy + (nb * sizeof(YRec) * G + 255) / 256 * 256;  // (counters)
    if (e == cudaSuccess) e = cudaMalloc(&ctx->xblock, ctx->xrec + 256);
    if (e == cudaSuccess) e = cudaMemset(ctx->xblock + ctx->xrec, 0, 256);
    if (e == cudaSuccess) {
      ctx->rec_all = (uint32_t*)ctx->xblock;
      ctx->zall = (double*)(ctx->xblock + ctx->xz);
      ctx->yall = (YRec*)(ctx->xblock + ctx->xy);
    }
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  ncclResult_t nr = ncclSuccess;
  if (e == cudaSuccess && cfg->nranks > 1 && !vgroup) {
    ncclUniqueId uid;
    memcpy(&uid, cfg->nccl_unique_id, sizeof(uid));
    nr = ncclCommInitRank(&ctx->comm, cfg->nranks, uid, cfg->rank);
    if (nr != ncclSuccess) ctx->comm = nullptr;
    if (nr == ncclSuccess && cfg->nranks <= kMaxPeers && cfg->exchange == 0) p2p_attach(ctx);
  }
  if (e != cudaSuccess || nr != ncclSuccess) {
    std::string msg = (e != cudaSuccess) ? std::string("init: ") + cudaGetErrorString(e)
                                         : std::string("init: ncclCommInitRank: ") + ncclGetErrorString(nr);
    cudaFree(ctx->rec_send);
    cudaFree(ctx->zsend);
    cudaFree(ctx->ysend);
    cudaFree(ctx->xblock);
    cudaFree(ctx->lz);
    cudaGetLastError();
    cudaFree(ctx->parts);
    cudaFree(ctx->pdec);
    cudaFree(ctx->counters);
    cudaFree(ctx->ndec);
    cudaFree(ctx->cpq);
    cudaFree(ctx->segsum);
  cudaFree(ctx->slices);
    cudaFree(ctx->slices);
    delete ctx;
    if (e == cudaSuccess) return fail(nullptr, COSINE_ERR_NCCL, msg);
    return fail(nullptr, e == cudaErrorMemoryAllocation ? COSINE_ERR_OUT_OF_MEMORY : COSINE_ERR_CUDA, msg);
  }
  *out = ctx;
  return COSINE_OK;
}

cosine_status_t cosine_verify_init(const cosine_config_t* cfg, cosine_ctx_t* out) {
  return init_impl(cfg, out, false);
}

cosine_status_t cosine_verify_init_vgroup(const cosine_config_t* cfgs, int32_t G, cosine_ctx_t* out) {
  if (!cfgs || !out || G < 2 || G > 32) return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "bad cfgs / out / G");
  for (int g = 0; g < G; ++g) out[g] = nullptr;
  for (int g = 0; g < G; ++g) {
    const cosine_config_t& c = cfgs[g];
    if (c.nranks != G || c.rank != g || c.vocab_size != cfgs[0].vocab_size ||
        c.vocab_begin != (g == 0 ? 0 : cfgs[g - 1].vocab_end) || (g == G - 1 && c.vocab_end != c.vocab_size) ||
        c.target_dtype != cfgs[0].target_dtype || c.draft_dtype != cfgs[0].draft_dtype ||
        c.draft_kind != cfgs[0].draft_kind || c.seed != cfgs[0].seed || c.max_batch != cfgs[0].max_batch ||
        c.max_draft_len != cfgs[0].max_draft_len || c.max_drafters != cfgs[0].max_drafters) {
      for (int h = 0; h < g; ++h) cosine_verify_destroy(out[h]);
      return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT,
                  "vgroup: cfgs[g] must be rank g of G with shards tiling [0, vocab_size) and equal settings");
    }
    const cosine_status_t s = init_impl(&c, &out[g], true);
    if (s != COSINE_OK) {
      for (int h = 0; h < g; ++h) cosine_verify_destroy(out[h]);
      out[g] = nullptr;
      return s;
    }
  }
  return COSINE_OK;
}

cosine_status_t cosine_verify_destroy(cosine_ctx_t ctx) {
  if (!ctx) return COSINE_OK;
  DeviceGuard dg(ctx->cfg.device);
  cudaDeviceSynchronize();
  cudaFree(ctx->parts);
  cudaFree(ctx->pdec);
  cudaFree(ctx->counters);
  cudaFree(ctx->ndec);
  cudaFree(ctx->cpq);
  cudaFree(ctx->segsum);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  cudaFree(ctx->lz);
  for (int g = 0; g < kMaxPeers; ++g)
    if (ctx->peer_block[g] && ctx->peer_block[g] != ctx->xblock && !ctx->vgroup) cudaIpcCloseMemHandle(ctx->peer_block[g]);
  cudaFree(ctx->rec_send);
  cudaFree(ctx->zsend);
  cudaFree(ctx->ysend);
  cudaFree(ctx->xblock);
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

int32_t cosine_exchange_mode(cosine_ctx_t ctx) {
  if (!ctx || ctx->cfg.nranks == 1) return 0;
  return ctx->vgroup ? 3 : (ctx->p2p ? 2 : 1);
}

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
  const CallDims P0 = call_dims(ctx, ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS ? temperature : 1.f);
  SplitParams S;
  memset(&S, 0, sizeof(S));
  S.mode = kSplitFuse;
  S.B = B; S.k = k; S.N = N;
  S.V = P0.V; S.ld_t = ld_q; S.ld_q = ld_q; S.ngroups = P0.ngroups; S.gfull = P0.gfull;
  S.k2f = P0.k2f; S.k2d = P0.k2d; S.greedy = 0; S.weight_mode = weight_mode; S.select = select_mode;
  S.draft = draft; S.target = draft; S.draft_tokens = draft_tokens; S.rids = request_ids; S.seed = P0.seed;
  S.step = step; S.status = status;
  S.fuse_tokens = fused_tokens; S.fuse_w = weights; S.fuse_sig = draft_norm; S.fused_q = fused_q; S.ld_fq = ld_fq;
  const int64_t units = (int64_t)B * k;
  fill_scratch(ctx, S, stats_chunks(ctx, units, S.ngroups));
  // the drafter rows stand in for the (absent) target rows of the statistics kernel, so it runs
  // with the drafters' dtype on both (stats_body, kSplitFuse)
  KernelSet ks;
  kernel_set(ctx->cfg.draft_dtype, ctx->cfg.draft_dtype, ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS, N, &ks);
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.gridDim = dim3((unsigned)(units * S.C), 1, 1);
  cudaError_t e = cudaLaunchKernelEx(&lc, ks.stats, S);
  lc.attrs = at;
  lc.numAttrs = 1;
  int launches = 1;
  if (e == cudaSuccess) {
    lc.gridDim = dim3((unsigned)units, 1, 1);
    e = cudaLaunchKernelEx(&lc, ks.fuse_decide, S);
    ++launches;
  }
  if (e == cudaSuccess && fused_q) {
    lc.gridDim = dim3((unsigned)(units * S.C), 1, 1);
    e = cudaLaunchKernelEx(&lc, ks.fuse_write_q, S);
    ++launches;
  }
  if (e == cudaSuccess) {
    lc.gridDim = dim3((unsigned)((B + kThreads - 1) / kThreads), 1, 1);
    e = cudaLaunchKernelEx(&lc, fuse_finish_kernel, S);
    ++launches;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("fuse_drafts kernels: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = launches;
  return COSINE_OK;
}

// Argument checks shared by cosine_verify_batch and cosine_verify_batch_vgroup.
static cosine_status_t check_verify(cosine_ctx_t ctx, int32_t B, int32_t k, int32_t N, const void* target_logits,
                                    int64_t ld_t, float temperature, const void* draft, int64_t ld_q,
                                    const int32_t* draft_tokens, const uint64_t* request_ids,
                                    cosine_weight_mode_t weight_mode, cosine_select_mode_t select_mode,
                                    int32_t* accept_len, int32_t* out_tokens, int32_t* status) {
  cosine_status_t s = check_common(ctx, B, k, N);
  if (s != COSINE_OK) return s;
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
  return COSINE_OK;
}

// The split-kernel parameters of a verify call (everything but the launch configuration).
static SplitParams make_split(cosine_ctx_t ctx, int32_t B, int32_t k, int32_t N, const void* target_logits,
                              int64_t ld_t, float temperature, const void* draft, int64_t ld_q,
                              const int32_t* draft_tokens, const int32_t* draft_len, const uint64_t* request_ids,
                              uint32_t step, cosine_weight_mode_t weight_mode, int32_t* accept_len,
                              int32_t* out_tokens, int32_t* status, const cosine_debug_t* debug,
                              cosine_select_mode_t select_mode = COSINE_SEL_ARGMAX) {
  const CallDims P = call_dims(ctx, temperature);
  SplitParams S;
  memset(&S, 0, sizeof(S));
  S.B = B; S.k = k; S.N = N;
  S.V = P.V; S.ld_t = ld_t; S.ld_q = ld_q; S.ngroups = P.ngroups; S.gfull = P.gfull;
  S.k2f = P.k2f; S.k2d = P.k2d; S.greedy = P.greedy; S.weight_mode = weight_mode; S.select = select_mode;
  S.target = target_logits; S.draft = draft; S.draft_tokens = draft_tokens; S.draft_len = draft_len;
  S.rids = request_ids; S.seed = P.seed; S.step = step;
  S.accept_len = accept_len; S.out_tokens = out_tokens; S.status = status;
  if (debug) S.dbg = *debug;
  return S;
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
  cosine_status_t s = check_verify(ctx, B, k, N, target_logits, ld_t, temperature, draft, ld_q, draft_tokens,
                                   request_ids, weight_mode, select_mode, accept_len, out_tokens, status);
  if (s != COSINE_OK) return s;
  if (B == 0) { ctx->last_launches = 0; return COSINE_OK; }
  if (ctx->vgroup) return fail(ctx, COSINE_ERR_UNSUPPORTED, "a vgroup context runs through cosine_verify_batch_vgroup");
  DeviceGuard dg(ctx->cfg.device);
  if (ctx->cfg.nranks > 1) {  // vocabulary-sharded (cosine_shard.cuh)
    if (select_mode != COSINE_SEL_ARGMAX)
      return fail(ctx, COSINE_ERR_UNSUPPORTED, "vocabulary sharding takes ARGMAX selection");
    SplitParams S = make_split(ctx, B, k, N, target_logits, ld_t, temperature, draft, ld_q, draft_tokens, draft_len,
                               request_ids, step, weight_mode, accept_len, out_tokens, status, debug);
    return launch_shard(ctx, (cudaStream_t)stream, S, ctx->cfg.target_dtype, ctx->cfg.draft_dtype,
                        ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS);
  }
  SplitParams S = make_split(ctx, B, k, N, target_logits, ld_t, temperature, draft, ld_q, draft_tokens, draft_len,
                             request_ids, step, weight_mode, accept_len, out_tokens, status, debug, select_mode);
  return launch_split(ctx, (cudaStream_t)stream, S, ctx->cfg.target_dtype, ctx->cfg.draft_dtype,
                      ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS, select_mode == COSINE_SEL_SAMPLE);
}

cosine_status_t cosine_verify_batch_vgroup(const cosine_ctx_t* ctxs, int32_t G, cosine_stream_t stream, int32_t B,
                                           int32_t k, int32_t N, const void* const* target_logits, int64_t ld_t,
                                           float temperature, const void* const* draft, int64_t ld_q,
                                           const int32_t* draft_tokens, const int32_t* draft_len,
                                           const uint64_t* request_ids, uint32_t step,
                                           cosine_weight_mode_t weight_mode, int32_t* const* accept_len,
                                           int32_t* const* out_tokens, int32_t* const* status, int32_t exchange) {
  if (!ctxs || G < 2 || !target_logits || !draft || !accept_len || !out_tokens || !status || exchange < 0 ||
      exchange > 1 || (exchange == 1 && G > kMaxPeers))
    return fail(nullptr, COSINE_ERR_INVALID_ARGUMENT, "vgroup: NULL argument or G < 2");
  for (int g = 0; g < G; ++g) {
    if (!ctxs[g] || !ctxs[g]->vgroup || ctxs[g]->cfg.nranks != G || ctxs[g]->cfg.rank != g)
      return fail(ctxs[g], COSINE_ERR_INVALID_ARGUMENT, "vgroup: ctxs[g] must be rank g of a G-context vgroup");
    cosine_status_t s = check_verify(ctxs[g], B, k, N, target_logits[g], ld_t, temperature, draft[g], ld_q,
                                     draft_tokens, request_ids, weight_mode, COSINE_SEL_ARGMAX, accept_len[g],
                                     out_tokens[g], status[g]);
    if (s != COSINE_OK) return s;
  }
  if (B == 0) return COSINE_OK;
  DeviceGuard dg(ctxs[0]->cfg.device);
  for (int g = 1; g < G; ++g)
    if (ctxs[g]->cfg.device != ctxs[0]->cfg.device)
      return fail(ctxs[g], COSINE_ERR_UNSUPPORTED, "vgroup: every context on one device");
  std::vector<SplitParams> S(G);
  for (int g = 0; g < G; ++g)
    S[g] = make_split(ctxs[g], B, k, N, target_logits[g], ld_t, temperature, draft[g], ld_q, draft_tokens, draft_len,
                      request_ids, step, weight_mode, accept_len[g], out_tokens[g], status[g], nullptr);
  const cosine_config_t& c = ctxs[0]->cfg;
  return launch_shard_vgroup(ctxs, G, (cudaStream_t)stream, S.data(), c.target_dtype, c.draft_dtype,
                             c.draft_kind == COSINE_DRAFT_LOGITS, exchange == 1);
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
  const CallDims P = call_dims(ctx, temperature);
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
  const CallDims P0 = call_dims(ctx, temperature);
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
  const int C = stats_chunks(ctx, units, S.ngroups);
  S.C = C;
  S.cg = (S.ngroups + C - 1) / C;
  KernelSet ks;
  kernel_set(ctx->cfg.target_dtype, ctx->cfg.draft_dtype, ctx->cfg.draft_kind == COSINE_DRAFT_LOGITS, N, &ks);
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
    e = cudaLaunchKernelEx(&lc, ks.stats, S);  // every node's rows, once
    if (e == cudaSuccess) {
      lc.gridDim = dim3((unsigned)((units + kWarps - 1) / kWarps), 1, 1);
      lc.attrs = at;
      lc.numAttrs = 1;
      e = cudaLaunchKernelEx(&lc, ks.tree_decide, T);
    }
  }
  if (e == cudaSuccess) {
    lc.gridDim = dim3((unsigned)B, 1, 1);
    lc.blockDim = dim3(kTreeBlock, 1, 1);
    lc.dynamicSmemBytes = (size_t)tree_walk_smem(nmax, (ngroups + tg - 1) / tg);
    cudaFuncAttributes fa;
    int optin = 0;
    e = cudaFuncGetAttributes(&fa, ks.tree_walk);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->cfg.device);
    if (e == cudaSuccess && fa.sharedSizeBytes + lc.dynamicSmemBytes > (size_t)optin) {
      ctx->last_launches = 2;
      return fail(ctx, COSINE_ERR_UNSUPPORTED, "vocabulary too wide for the tree walk's shared memory");
    }
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ks.tree_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lc.dynamicSmemBytes);
#ifdef COSINE_TRACE
    T.S.trace = cosine_trace_buffer((size_t)B * 16);
#endif
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&lc, ks.tree_walk, T);
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
  const CallDims P0 = call_dims(ctx, temperature);
  SplitParams S;
  memset(&S, 0, sizeof(S));
  S.mode = kSplitSample;
  S.B = B; S.k = 1; S.N = draft_rows ? N : 0;
  S.V = P0.V; S.ld_t = ld_t; S.ld_q = ld_q; S.ngroups = P0.ngroups; S.gfull = P0.gfull;
  S.k2f = P0.k2f; S.k2d = P0.k2d; S.greedy = P0.greedy; S.weight_mode = COSINE_W_CONF;
  S.target = target_rows; S.draft = draft_rows; S.rids = request_ids; S.seed = P0.seed; S.step = step;
  S.row_max = row_max; S.row_sumexp = row_sumexp; S.w_in = weights; S.norm_in = draft_norm;
  S.node_ids = node_ids; S.out_token = out_token; S.status = status;
  fill_scratch(ctx, S, stats_chunks(ctx, B, S.ngroups));
  if ((size_t)S.B * (size_t)S.nseg > ctx->segsum_cap)
    return fail(ctx, COSINE_ERR_INVALID_ARGUMENT, "segment scratch too small");
  KernelSet ks;
  kernel_set(ctx->cfg.target_dtype, ctx->cfg.draft_dtype, false, std::max(N, 1), &ks);
  cudaLaunchConfig_t lc;
  memset(&lc, 0, sizeof(lc));
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.gridDim = dim3((unsigned)((int64_t)B * S.C), 1, 1);
  cudaError_t e = cudaLaunchKernelEx(&lc, ks.stats, S);  // row statistics and validity checks
  lc.attrs = at;
  lc.numAttrs = 1;
  if (e == cudaSuccess) {
    lc.gridDim = dim3((unsigned)((B + kWarps - 1) / kWarps), 1, 1);
    e = cudaLaunchKernelEx(&lc, ks.sample_prep, S);
  }
  if (e == cudaSuccess) {
    lc.gridDim = dim3((unsigned)(B * S.spr), 1, 1);
    e = cudaLaunchKernelEx(&lc, ks.resample, S);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaMemsetAsync(ctx->counters, 0, ctx->counters_bytes, (cudaStream_t)stream);
    cudaGetLastError();
    ctx->last_launches = 0;
    return fail(ctx, COSINE_ERR_CUDA, std::string("sample_residual kernels: ") + cudaGetErrorString(e));
  }
  ctx->last_launches = 3;
  return COSINE_OK;
}

}  // extern "C"

#ifdef COSINE_TRACE
extern "C" size_t cosine_trace_read(unsigned long long* host, size_t n) { return cosine_trace_copy(host, n); }
#endif
