// cosine_kernels.cuh — device building blocks of the sm_100a verification kernels.
//
// Nothing here is shared with the CPU oracle (oracle/): this is an independent
// implementation of the same paper passages.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cosine {

constexpr int kThreads = 256;  // 8 warps per CTA
constexpr int kWarps = kThreads / 32;
constexpr int kMaxN = 8;       // drafters
constexpr int kMaxC = 16;      // CTAs per cluster (one (request, position) unit per cluster)
constexpr int kGroup = 8;      // vocabulary elements per group (one 16-byte bf16 vector)
constexpr int kNoReject = 0x7fffffff;
constexpr int kSegGroups = 512;  // solo sampling: groups per warp-owned segment
constexpr int kTileGroups = 256;  // sampling segment: groups per warp
constexpr int kTileElems = kTileGroups * 8;
constexpr int kMaxSeg = 256;     // segments per row (segment size grows beyond)
constexpr float kNegBig = -3.402823466e+38f;  // running-max seed: finite so that -inf - m = -inf

// Philox tags (header: ACCEPT = 0, SAMPLE = 1, FUSE = 2).
constexpr uint32_t kTagAccept = 0, kTagSample = 1, kTagFuse = 2;

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11) -> 24-bit uniform (readings #8, #9)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double philox_u24(uint64_t seed, uint64_t rid, uint32_t node,
                                             uint32_t step, uint32_t tag) {
  uint32_t x0 = (uint32_t)rid, x1 = (uint32_t)(rid >> 32), x2 = node, x3 = (step << 4) | tag;
  uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t a_hi = __umulhi(0xD2511F53u, x0), a_lo = 0xD2511F53u * x0;
    const uint32_t b_hi = __umulhi(0xCD9E8D57u, x2), b_lo = 0xCD9E8D57u * x2;
    const uint32_t y0 = b_hi ^ x1 ^ key0;
    const uint32_t y2 = a_hi ^ x3 ^ key1;
    x0 = y0; x1 = b_lo; x2 = y2; x3 = a_lo;
    key0 += 0x9E3779B9u;
    key1 += 0xBB67AE85u;
  }
  return (double)(x0 >> 8) * (1.0 / 16777216.0);
}

// ---------------------------------------------------------------------------
// Loads: 128-bit read-only streaming loads, 8 elements per group
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <typename T>
struct Group;

template <>
struct Group<__nv_bfloat16> {
  uint4 a;
  __device__ __forceinline__ void load(const __nv_bfloat16* row, int64_t g) {
    a = ld_stream(row + g * kGroup);
  }
  __device__ __forceinline__ void load_s(const __nv_bfloat16* srow, int g) {  // shared memory
    a = *reinterpret_cast<const uint4*>(srow + g * kGroup);
  }
  __device__ __forceinline__ void unpack(float f[8]) const {
    f[0] = __uint_as_float(a.x << 16); f[1] = __uint_as_float(a.x & 0xffff0000u);
    f[2] = __uint_as_float(a.y << 16); f[3] = __uint_as_float(a.y & 0xffff0000u);
    f[4] = __uint_as_float(a.z << 16); f[5] = __uint_as_float(a.z & 0xffff0000u);
    f[6] = __uint_as_float(a.w << 16); f[7] = __uint_as_float(a.w & 0xffff0000u);
  }
  __device__ __forceinline__ bool any_sign() const {
    return ((a.x | a.y | a.z | a.w) & 0x80008000u) != 0u;
  }
  __device__ __forceinline__ void zero() { a = make_uint4(0u, 0u, 0u, 0u); }
};

template <>
struct Group<float> {
  uint4 a, b;
  __device__ __forceinline__ void load(const float* row, int64_t g) {
    a = ld_stream(row + g * kGroup);
    b = ld_stream(row + g * kGroup + 4);
  }
  __device__ __forceinline__ void load_s(const float* srow, int g) {  // shared memory
    a = *reinterpret_cast<const uint4*>(srow + g * kGroup);
    b = *reinterpret_cast<const uint4*>(srow + g * kGroup + 4);
  }
  __device__ __forceinline__ void unpack(float f[8]) const {
    f[0] = __uint_as_float(a.x); f[1] = __uint_as_float(a.y);
    f[2] = __uint_as_float(a.z); f[3] = __uint_as_float(a.w);
    f[4] = __uint_as_float(b.x); f[5] = __uint_as_float(b.y);
    f[6] = __uint_as_float(b.z); f[7] = __uint_as_float(b.w);
  }
  __device__ __forceinline__ bool any_sign() const {
    return ((a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) & 0x80000000u) != 0u;
  }
  __device__ __forceinline__ void zero() { a = b = make_uint4(0u, 0u, 0u, 0u); }
};

__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f(float x) { return x; }

// The last (partial) group: elements >= V read as `pad`.
template <typename T>
__device__ __forceinline__ void load_partial(const T* row, int64_t g, int64_t V, float pad,
                                             float f[8]) {
#pragma unroll
  for (int e = 0; e < kGroup; ++e) {
    const int64_t v = g * kGroup + e;
    f[e] = (v < V) ? to_f(row[v]) : pad;
  }
}

template <typename T>
__device__ __forceinline__ float load_one(const T* row, int64_t v) {
  return to_f(row[v]);
}

__device__ __forceinline__ float max8(const float f[8]) {
  return fmaxf(fmaxf(fmaxf(f[0], f[1]), fmaxf(f[2], f[3])),
               fmaxf(fmaxf(f[4], f[5]), fmaxf(f[6], f[7])));
}
__device__ __forceinline__ float sum8(const float f[8]) {
  return ((f[0] + f[1]) + (f[2] + f[3])) + ((f[4] + f[5]) + (f[6] + f[7]));
}

// ---------------------------------------------------------------------------
// Warp reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
// (value, index) argmax with the lowest index on ties; idx < 0 means "none".
__device__ __forceinline__ void warp_argmax(float& v, int64_t& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (oi >= 0 && (idx < 0 || ov > v || (ov == v && oi < idx))) { v = ov; idx = oi; }
  }
}

// ---------------------------------------------------------------------------
// Device counters between CTAs: release arrivals (the CTA's writes, ordered before by a barrier,
// become visible before the count: the red/atom's release is cumulative) and acquire waits
// (ld.acquire).  A plain __threadfence (fence.sc + L1 invalidate) + atomicAdd costs the
// arriving CTA ~1 us more before it can retire.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void red_release_add(int32_t* p, int32_t v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t atom_acq_rel_add(int32_t* p, int32_t v) {
  int32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ---------------------------------------------------------------------------
// Cluster barrier halves and mbarriers (PTX ISA: barrier.cluster, mbarrier, mapa)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Arrive (release, cluster scope) on the mbarrier at the same smem offset in CTA `rank`.
__device__ __forceinline__ void mbar_remote_arrive(uint64_t* bar, uint32_t rank) {
  uint32_t raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Bulk async copies (TMA, non-tensor): global -> this CTA's shared memory, completion counted in
// bytes on an mbarrier (PTX ISA: cp.async.bulk, mbarrier.expect_tx).
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace cosine
