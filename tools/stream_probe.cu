// stream_probe.cu — HBM read-bandwidth probes for the verification access pattern (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe tools/stream_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint4 ldnc(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float s8(uint4 a) {
  return __uint_as_float(a.x << 16) + __uint_as_float(a.x & 0xffff0000u) + __uint_as_float(a.y << 16) +
         __uint_as_float(a.y & 0xffff0000u) + __uint_as_float(a.z << 16) + __uint_as_float(a.z & 0xffff0000u) +
         __uint_as_float(a.w << 16) + __uint_as_float(a.w & 0xffff0000u);
}

// (a) flat grid-stride read, U loads in flight per thread
template <int U>
__global__ void flat(const uint4* __restrict__ p, size_t n, float* out) {
  float acc = 0.f;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldnc(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += s8(v[u]);
  }
  for (; i < n; i += stride) acc += s8(ldnc(p + i));
  if (acc == 123.f) out[0] = acc;
}

// (b) the verify pattern: unit = R rows of V bf16; CTA (unit, chunk) streams its chunk of all rows
template <int R>
__global__ void rows(const uint4* __restrict__ p, int64_t ld16, int64_t nvec, int C, float* out) {
  const int64_t unit = blockIdx.x / C;
  const int r = blockIdx.x % C;
  const int64_t cv = (nvec + C - 1) / C;
  const int64_t b0 = r * cv, b1 = min(nvec, b0 + cv);
  const uint4* base = p + unit * R * ld16;
  float acc = 0.f;
  for (int64_t v = b0 + threadIdx.x; v < b1; v += blockDim.x) {
    uint4 x[R];
#pragma unroll
    for (int q = 0; q < R; ++q) x[q] = ldnc(base + q * ld16 + v);
#pragma unroll
    for (int q = 0; q < R; ++q) acc += s8(x[q]);
  }
  if (acc == 123.f) out[0] = acc;
}

// (c) same pattern, 2 groups per row in flight
template <int R>
__global__ void rows2(const uint4* __restrict__ p, int64_t ld16, int64_t nvec, int C, float* out) {
  const int64_t unit = blockIdx.x / C;
  const int r = blockIdx.x % C;
  const int64_t cv = (nvec + C - 1) / C;
  const int64_t b0 = r * cv, b1 = min(nvec, b0 + cv);
  const uint4* base = p + unit * R * ld16;
  float acc = 0.f;
  int64_t v = b0 + threadIdx.x;
  for (; v + blockDim.x < b1; v += 2 * blockDim.x) {
    uint4 x[2 * R];
#pragma unroll
    for (int q = 0; q < R; ++q) { x[2 * q] = ldnc(base + q * ld16 + v); x[2 * q + 1] = ldnc(base + q * ld16 + v + blockDim.x); }
#pragma unroll
    for (int q = 0; q < 2 * R; ++q) acc += s8(x[q]);
  }
  for (; v < b1; v += blockDim.x)
    for (int q = 0; q < R; ++q) acc += s8(ldnc(base + q * ld16 + v));
  if (acc == 123.f) out[0] = acc;
}


__device__ __forceinline__ float ex2f_(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ void unpack8(uint4 a, float f[8]) {
  f[0] = __uint_as_float(a.x << 16); f[1] = __uint_as_float(a.x & 0xffff0000u);
  f[2] = __uint_as_float(a.y << 16); f[3] = __uint_as_float(a.y & 0xffff0000u);
  f[4] = __uint_as_float(a.z << 16); f[5] = __uint_as_float(a.z & 0xffff0000u);
  f[6] = __uint_as_float(a.w << 16); f[7] = __uint_as_float(a.w & 0xffff0000u);
}
// (d) verify-like compute: row 0 online softmax (FFMA form), rows 1..R-1 sums; PF = prefetch depth
template <int R, int PF, bool kFFMA>
__global__ void __launch_bounds__(256) vcompute(const uint4* __restrict__ p, int64_t ld16, int64_t nvec, int C, float k2, float* out) {
  const int64_t unit = blockIdx.x / C;
  const int r = blockIdx.x % C;
  const int64_t cv = (nvec + C - 1) / C;
  const int64_t b0 = r * cv, b1 = min(nvec, b0 + cv);
  const uint4* base = p + unit * R * ld16;
  float m = -3.0e38f, mk = -3.0e38f * k2, s = 0.f, ds[R];
  for (int q = 0; q < R; ++q) ds[q] = 0.f;
  uint4 buf[PF][R];
  int64_t v = b0 + threadIdx.x;
#pragma unroll
  for (int f = 0; f < PF; ++f)
#pragma unroll
    for (int q = 0; q < R; ++q) if (v + f * blockDim.x < b1) buf[f][q] = ldnc(base + q * ld16 + v + f * blockDim.x);
  for (; v < b1; v += blockDim.x) {
    uint4 cur[R];
#pragma unroll
    for (int q = 0; q < R; ++q) cur[q] = buf[0][q];
#pragma unroll
    for (int f = 0; f + 1 < PF; ++f)
#pragma unroll
      for (int q = 0; q < R; ++q) buf[f][q] = buf[f + 1][q];
    const int64_t vn = v + PF * blockDim.x;
#pragma unroll
    for (int q = 0; q < R; ++q) if (vn < b1) buf[PF - 1][q] = ldnc(base + q * ld16 + vn);
    float f[8];
    unpack8(cur[0], f);
    float gm = fmaxf(fmaxf(fmaxf(f[0], f[1]), fmaxf(f[2], f[3])), fmaxf(fmaxf(f[4], f[5]), fmaxf(f[6], f[7])));
    if (gm > m) { s *= ex2f_((m - gm) * k2); m = gm; mk = m * k2; }
    float e[8];
    if (kFFMA) {
#pragma unroll
      for (int i = 0; i < 8; ++i) e[i] = ex2f_(fmaf(f[i], k2, -mk));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) e[i] = ex2f_((f[i] - m) * k2);
    }
    s += ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
#pragma unroll
    for (int q = 1; q < R; ++q) {
      unpack8(cur[q], f);
      ds[q] += ((f[0] + f[1]) + (f[2] + f[3])) + ((f[4] + f[5]) + (f[6] + f[7]));
    }
  }
  float acc = s + m;
  for (int q = 1; q < R; ++q) acc += ds[q];
  if (acc == 123.f) out[0] = acc;
}

int main() {
  const int64_t V = 128256, nvec = V / 8, units = 2304;
  const int R = 5;
  const size_t bytes = (size_t)units * R * V * 2;
  void* buf;
  float* out;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(buf, 0, bytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    const int it = 20;
    for (int w = 0; w < it; ++w) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t er = cudaGetLastError();
    printf("%-40s %8.1f us  %7.1f GB/s  %s\n", name, 1e3 * ms / it, bytes / (1e6 * ms / it), cudaGetErrorString(er));
  };
  const size_t n16 = bytes / 16;
  for (int C : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "vcompute PF=1 sub C=%d", C);
    timeit(nm, [&] { vcompute<5, 1, false><<<(unsigned)(units * C), 256>>>((const uint4*)buf, V / 8, nvec, C, 1.4427f, out); });
    snprintf(nm, 64, "vcompute PF=1 ffma C=%d", C);
    timeit(nm, [&] { vcompute<5, 1, true><<<(unsigned)(units * C), 256>>>((const uint4*)buf, V / 8, nvec, C, 1.4427f, out); });
    snprintf(nm, 64, "vcompute PF=2 ffma C=%d", C);
    timeit(nm, [&] { vcompute<5, 2, true><<<(unsigned)(units * C), 256>>>((const uint4*)buf, V / 8, nvec, C, 1.4427f, out); });
    snprintf(nm, 64, "vcompute PF=3 ffma C=%d", C);
    timeit(nm, [&] { vcompute<5, 3, true><<<(unsigned)(units * C), 256>>>((const uint4*)buf, V / 8, nvec, C, 1.4427f, out); });
  }
  timeit("flat U=1 grid=148*8 x256", [&] { flat<1><<<148 * 8, 256>>>((const uint4*)buf, n16, out); });
  timeit("flat U=4 grid=148*8 x256", [&] { flat<4><<<148 * 8, 256>>>((const uint4*)buf, n16, out); });
  timeit("flat U=8 grid=148*4 x256", [&] { flat<8><<<148 * 4, 256>>>((const uint4*)buf, n16, out); });
  timeit("flat U=4 grid=148*16 x256", [&] { flat<4><<<148 * 16, 256>>>((const uint4*)buf, n16, out); });
  for (int C : {1, 2, 4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "rows R=5 C=%d x256", C);
    timeit(nm, [&] { rows<5><<<(unsigned)(units * C), 256>>>((const uint4*)buf, V / 8, nvec, C, out); });
    snprintf(nm, 64, "rows2 R=5 C=%d x256", C);
    timeit(nm, [&] { rows2<5><<<(unsigned)(units * C), 256>>>((const uint4*)buf, V / 8, nvec, C, out); });
    snprintf(nm, 64, "rows R=5 C=%d x512", C);
    timeit(nm, [&] { rows<5><<<(unsigned)(units * C), 512>>>((const uint4*)buf, V / 8, nvec, C, out); });
  }
  return 0;
}
