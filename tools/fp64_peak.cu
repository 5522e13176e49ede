// FP64 peak microbenchmark for the roofline denominator (B200 has no FP64
// figure in MEASURED_PEAKS.json).  Measures DMMA (mma.sync f64 shapes) and
// DFMA throughput with many independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 - i;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_chains(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
static float time_kernel(K kern, int blocks, int threads, double* out, int iters, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  size_t fr, tot; cudaMemGetInfo(&fr, &tot);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"smem_optin\": %zu, \"mem_total\": %zu, \"mem_free\": %zu, \"l2\": %d}\n",
         p.name, sms, (size_t)p.sharedMemPerBlockOptin, tot, fr, p.l2CacheSize);
  double* out; CK(cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024));
  const int iters = 4096;
  for (int wpb : {4, 8, 16}) {
    int threads = 32 * wpb;
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      float ms = time_kernel(dmma_m8n8k4<8>, blocks, threads, out, iters, 5);
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * (double)wpb);
      printf("{\"op\": \"dmma_m8n8k4\", \"warps_per_block\": %d, \"blocks\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
             wpb, blocks, ms, flops / ms / 1e9);
      ms = time_kernel(dmma_m16n8k16<4>, blocks, threads, out, iters / 4, 5);
      flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * (blocks * (double)wpb);
      printf("{\"op\": \"dmma_m16n8k16\", \"warps_per_block\": %d, \"blocks\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
             wpb, blocks, ms, flops / ms / 1e9);
      ms = time_kernel(dfma_chains<16>, blocks, threads, out, iters, 5);
      flops = 2.0 * 16.0 * iters * (blocks * (double)threads);
      printf("{\"op\": \"dfma\", \"warps_per_block\": %d, \"blocks\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
             wpb, blocks, ms, flops / ms / 1e9);
    }
  }
  // sustained: DMMA back to back for ~4 s
  {
    int blocks = sms * 2, threads = 256;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int it2 = 65536; int reps = 0; float tot_ms = 0;
    cudaEventRecord(e0);
    while (tot_ms < 4000.f) {
      dmma_m8n8k4<8><<<blocks, threads>>>(out, it2);
      ++reps;
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&tot_ms, e0, e1);
    }
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * it2 * (blocks * 8.0) * reps;
    printf("{\"op\": \"dmma_m8n8k4_sustained\", \"seconds\": %.2f, \"tflops\": %.2f}\n", tot_ms / 1e3, flops / tot_ms / 1e9);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
