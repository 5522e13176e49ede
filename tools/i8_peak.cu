// Tensor-core issue-rate microbenchmark for the int8 roofline denominator
// (MEASURED_PEAKS.json has bf16 only): one thread per CTA issues back-to-back
// tcgen05.mma (M = 128, N in {64, 128, 256}, K = 32 bytes) on a resident
// shared-memory tile, no loads in the loop; kind::i8 next to kind::f8f6f4
// (e4m3) and kind::f16 (bf16) on the same harness.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/i8_peak.cu -o tools/i8_peak
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(unsigned saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
template <int KIND>
__device__ __forceinline__ void mma(unsigned tmem_d, uint64_t da, uint64_t db, unsigned idesc, unsigned acc) {
  if (KIND == 0)
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}"
                 ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
  else if (KIND == 1)
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}"
                 ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                 ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
}

template <int KIND, int N>
__global__ void __launch_bounds__(128, 1) peak_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ unsigned slot;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x) ((unsigned*)smem)[i] = 0x01010101u * (i & 3);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = slot;
  if (threadIdx.x == 32) {
    // c_format: S32 (2) for i8, F32 (1) otherwise; a/b format: int8 signed (1), e4m3 (0), bf16 (1)
    const unsigned cf = KIND == 0 ? 2u : 1u, ab = KIND == 1 ? 0u : 1u;
    const unsigned idesc = (cf << 4) | (ab << 7) | (ab << 10) | ((unsigned)(N >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
    const unsigned a0 = smem_u32(smem), b0 = a0 + 128 * 128;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 8; ++u)   // 4 K steps of the 128-byte rows, two accumulators
        mma<KIND>(tmem + (u & 1) * 256 * (N <= 256), desc_sw128(a0 + (u >> 1) * 32), desc_sw128(b0 + (u >> 1) * 32), idesc,
                  1u);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(smem_u32(&bar)) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

template <int KIND, int N>
static void run(const char* name, int kbytes_per_mma_elems) {
  const int iters = 20000, grid = 148;
  long long* dc;
  CK(cudaMalloc(&dc, grid * 8));
  const int smem = (128 + N) * 128 + 2048;
  CK(cudaFuncSetAttribute(peak_kernel<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  peak_kernel<KIND, N><<<grid, 128, smem>>>(100, dc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  peak_kernel<KIND, N><<<grid, 128, smem>>>(iters, dc);
  CK(cudaEventRecord(e1));
  CK(cudaDeviceSynchronize());
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  long long hc[148];
  CK(cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost));
  const double mmas = (double)iters * 8;
  const double macs_per_mma = 128.0 * N * kbytes_per_mma_elems;   // K elements per instruction
  const double tops = 2.0 * mmas * macs_per_mma * grid / (ms * 1e-3) * 1e-12;
  printf("%-10s N=%3d: %.3f ms, %.1f cycles per MMA (SM 0), %.2f dense T(FL)OP/s on %d SMs, clock ~%.2f GHz\n", name, N, ms,
         hc[0] / mmas, tops, grid, hc[0] / (ms * 1e-3) * 1e-9);
  cudaFree(dc);
}

int main() {
  run<0, 64>("int8", 32);  run<0, 128>("int8", 32);  run<0, 256>("int8", 32);
  run<1, 64>("fp8 e4m3", 32); run<1, 128>("fp8 e4m3", 32); run<1, 256>("fp8 e4m3", 32);
  run<2, 64>("bf16", 16);  run<2, 128>("bf16", 16);  run<2, 256>("bf16", 16);
  return 0;
}
