// Dependent-chain latency of FP64 operations on one thread (cycles per op).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double seed, int iters) {
  double a = seed, b = seed * 0.5 + 1.0;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, 0.999999, 1e-9);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) b = b * 1.0000001;
  t1 = clock64();
  cyc[1] = t1 - t0;
  // rsqrt chain
  double c = seed + 2.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) c = rsqrt(c) + 1.5;
  t1 = clock64();
  cyc[2] = t1 - t0;
  // sqrt chain
  double d = seed + 3.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = sqrt(d) + 1.5;
  t1 = clock64();
  cyc[3] = t1 - t0;
  // division chain
  double e = seed + 4.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) e = 3.0 / e + 1.0;
  t1 = clock64();
  cyc[4] = t1 - t0;
  // float rsqrt + 2 Newton steps in fp64 (full precision rsqrt)
  double f = seed + 2.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double y = (double)rsqrtf((float)f);
    const double h = 0.5 * f;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    f = y + 1.5;
  }
  t1 = clock64();
  cyc[5] = t1 - t0;
  // DADD chain
  double g = seed;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) g = g + 1e-9;
  t1 = clock64();
  cyc[6] = t1 - t0;
  // shfl of a double (two 32-bit shuffles) chain
  double h = seed;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) h = __shfl_sync(0xffffffffu, h, (threadIdx.x + 1) & 31) + 1e-9;
  t1 = clock64();
  cyc[7] = t1 - t0;
  out[0] = a + b + c + d + e + f + g + h;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 8);
  const int iters = 4096;
  lat<<<1, 32>>>(out, cyc, 1.0, iters);
  lat<<<1, 32>>>(out, cyc, 1.0, iters);
  long long h[8];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[8] = {"DFMA", "DMUL", "rsqrt(double)", "sqrt(double)", "div(double)", "rsqrtf+2 Newton (fp64)", "DADD", "shfl double + DADD"};
  for (int i = 0; i < 8; ++i) printf("%-26s %7.1f cycles/op\n", names[i], (double)h[i] / iters);
  return 0;
}
