// Shared helpers for the CIRR sm_100a kernels: complex128 as double2
// (interleaved re/im, the torch complex128 layout), DMMA fragment wrappers,
// warp/block reductions and the C-ABI error convention.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "cirr.h"

typedef double2 cplx;

#define CIRR_API extern "C" __attribute__((visibility("default")))

// Every C-ABI entry returns 0 on success or a cudaError_t value (> 0);
// argument errors return CIRR_EINVAL.

// Host-side count of kernels this library has launched (cirr_launch_count).
extern long long g_cirr_launches;
inline void cirr_note_launch() { __atomic_fetch_add(&g_cirr_launches, 1, __ATOMIC_RELAXED); }

// Per-stream pair of device ints {next tile, finished CTAs} for the dynamic
// tile scheduler of the persistent GEMM (gemm.cu); zero between launches.
int* cirr_tile_counter(cudaStream_t stream);

// Stream-ordered scratch (cudaMallocAsync).  When the pool cannot grow -- the
// caller's allocator (PyTorch's caching allocator) holds the rest of HBM --
// the handler set by cirr_set_oom_handler runs (it releases that cache) and the
// allocation is retried once.
cudaError_t cirr_malloc_async(void** p, size_t bytes, cudaStream_t stream);

// Cap on the CTAs of the cooperative latency-bound kernels (0 = whole GPU);
// set by cirr_set_coop_ctas so they can run beside the bulk GEMMs.
extern int g_cirr_coop_cap;
// Cap on the CTAs of the persistent TMA GEMM (0 = every SM); set by
// cirr_set_gemm_ctas so latency-bound kernels on other streams find free SMs.
extern int g_cirr_gemm_cap;

#define CIRR_CHECK_LAUNCH()                              \
  do {                                                   \
    cirr_note_launch();                                  \
    cudaError_t _e = cudaGetLastError();                 \
    if (_e != cudaSuccess) return (int)_e;               \
  } while (0)

#define CIRR_TRY(expr)                                   \
  do {                                                   \
    int _r = (expr);                                     \
    if (_r != 0) return _r;                              \
  } while (0)

__host__ __device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return cmk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ cplx cconj(cplx a) { return cmk(a.x, -a.y); }
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return cmk(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
__host__ __device__ __forceinline__ double cabs1(cplx a) { return fabs(a.x) + fabs(a.y); }
// a * conj(b)
__host__ __device__ __forceinline__ cplx cmulc(cplx a, cplx b) {
  return cmk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// conj(a) * b
__host__ __device__ __forceinline__ cplx cconjmul(cplx a, cplx b) {
  return cmk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
// acc += a*b
__device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc -= a*b
__device__ __forceinline__ void cfms(cplx& acc, cplx a, cplx b) {
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
// Smith's algorithm for a / b
__host__ __device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, d = b.x + b.y * r;
    return cmk((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  } else {
    double r = b.x / b.y, d = b.y + b.x * r;
    return cmk((a.x * r + a.y) / d, (a.y * r - a.x) / d);
  }
}
__host__ __device__ __forceinline__ cplx crecip(cplx b) { return cdiv(cmk(1.0, 0.0), b); }
__host__ __device__ __forceinline__ double cabs(cplx a) { return hypot(a.x, a.y); }

// D(8x8, 2 per lane) += A(8x4, 1 per lane, row) * B(4x8, 1 per lane, col).
// Lane l holds A[l/4][l%4], B[l%4][l/4], C[l/4][2*(l%4)+{0,1}].  SASS: DMMA.8x8x4.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; `red` must hold >= 32 doubles; all threads get the result.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (wid == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  t = red[0];
  return t;
}
__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : -1.0;
  if (wid == 0) t = warp_max(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  t = red[0];
  return t;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Software grid barrier for cooperative launches (all CTAs co-resident).
// Two-level: CTAs arrive on one of ceil(G/16) group counters, the last of a
// group arrives on the top counter, the last overall bumps the generation --
// no single L2 address sees more than 16 atomics per barrier.  Every counter
// sits on its own 128-byte line: bar[0] generation, bar[32] top counter,
// bar[64 + 32*g] group g.  Needs (64 + 32*ceil(G/16)) * 4 bytes, zeroed.
constexpr int GB_GROUP = 16;
__host__ __device__ constexpr long long grid_barrier_bytes(int nblocks) {
  return (64LL + 32LL * ((nblocks + GB_GROUP - 1) / GB_GROUP)) * 4;
}
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar;
    const unsigned gen = *vgen;
    const unsigned g = blockIdx.x / GB_GROUP;
    const unsigned ngroups = (nblocks + GB_GROUP - 1) / GB_GROUP;
    const unsigned gsize = min((unsigned)GB_GROUP, nblocks - g * GB_GROUP);
    unsigned* gcnt = bar + 64 + 32 * g;
    __threadfence();
    if (atomicAdd(gcnt, 1u) == gsize - 1) {
      *gcnt = 0;
      __threadfence();
      if (atomicAdd(bar + 32, 1u) == ngroups - 1) {
        bar[32] = 0;
        __threadfence();
        atomicAdd(bar, 1u);
      }
    }
    while (*vgen == gen) { __nanosleep(20); }
    __threadfence();
  }
  __syncthreads();
}
