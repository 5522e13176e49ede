// Cost of the software grid barrier (common.cuh) with SC vs acq_rel fences.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2511_01927_b200/csrc -o tools/gridbar_bench tools/gridbar_bench.cu
#include <cstdio>
#include "common.cuh"
long long g_cirr_launches = 0;
int g_cirr_coop_cap = 0;

__device__ __forceinline__ void grid_barrier_ar(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar;
    const unsigned gen = *vgen;
    const unsigned g = blockIdx.x / GB_GROUP;
    const unsigned ngroups = (nblocks + GB_GROUP - 1) / GB_GROUP;
    const unsigned gsize = min((unsigned)GB_GROUP, nblocks - g * GB_GROUP);
    unsigned* gcnt = bar + 64 + 32 * g;
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (atomicAdd(gcnt, 1u) == gsize - 1) {
      *gcnt = 0;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (atomicAdd(bar + 32, 1u) == ngroups - 1) {
        bar[32] = 0;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        atomicAdd(bar, 1u);
      }
    }
    while (*vgen == gen) { __nanosleep(20); }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

template <int V>
__global__ void bench(unsigned* bar, int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (V == 0) grid_barrier(bar, gridDim.x);
    else grid_barrier_ar(bar, gridDim.x);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[V] = clock64() - t0;
}

int main() {
  unsigned* bar; long long* out;
  cudaMalloc(&bar, 65536); cudaMalloc(&out, 16);
  for (int grid : {148, 296}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(bar, 0, 65536);
      int iters = 2000;
      void* a0[] = {&bar, &iters, &out};
      cudaLaunchCooperativeKernel((void*)bench<0>, grid, 256, a0, 0, 0);
      cudaMemset(bar, 0, 65536);
      cudaLaunchCooperativeKernel((void*)bench<1>, grid, 256, a0, 0, 0);
      cudaDeviceSynchronize();
    }
    long long h[2];
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("grid %d: SC fence %.0f cycles/barrier, acq_rel fence %.0f cycles/barrier (%s)\n", grid, h[0] / 2000.0,
           h[1] / 2000.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
