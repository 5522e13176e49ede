// Cycles per step of the QR front recurrence alone (one warp, registers only),
// with three rsqrt variants.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2511_01927_b200/csrc
#include <cstdio>
#include "common.cuh"

template <int V>
__device__ __forceinline__ double rs(double a) {
  if (V == 0) return rsqrt(a);
  // MUFU.RSQ64H seed + 2 Newton steps, no special-case path (a > 0, normal)
  double y;
  asm("{.reg .f32 f; .reg .f64 t; cvt.rn.f32.f64 f, %1; rsqrt.approx.ftz.f32 f, f; cvt.f64.f32 %0, f;}" : "=d"(y) : "d"(a));
  const double h = 0.5 * a;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  if (V == 2) y = y * fma(-h * y, y, 1.5);
  return y;
}

template <int V>
__global__ void front(cplx* out, long long* cyc, int steps, cplx tcar, cplx u, cplx v) {
  cplx x = cmk(0.3, 0.1), y = cmk(0.2, -0.4), d = cmk(1.0, 0.5), e = cmk(0.7, 0.1);
  long long t0 = clock64();
  for (int m = 0; m < steps; ++m) {
    const double nx2 = cabs2(x), ny2 = cabs2(y);
    double c; cplx sn, r;
    const double ix = rs<V>(nx2);
    const double inv = rs<V>(nx2 + ny2);
    c = nx2 * ix * inv;
    const cplx ph = cscale(x, ix);
    sn = cscale(cmul(ph, cconj(y)), inv);
    r = cscale(ph, (nx2 + ny2) * inv);
    const cplx snc = cconj(sn);
    const cplx A0 = cadd(cscale(d, c), cmul(sn, e)), B0 = csub(cscale(e, c), cmul(snc, d));
    const cplx A1 = cadd(cscale(tcar, c), cmul(sn, u)), B1 = csub(cscale(u, c), cmul(snc, tcar));
    const cplx hmm = cadd(cscale(A0, c), cmul(snc, A1));
    const cplx xn = cadd(cscale(B0, c), cmul(snc, B1)), dn = csub(cscale(B1, c), cmul(sn, B0));
    const cplx yn = cmul(snc, v);
    const cplx en = cscale(v, c);
    x = cadd(xn, cscale(r, 1e-3)); y = cadd(yn, cscale(hmm, 1e-3)); d = dn; e = en;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[V] = t1 - t0; out[V] = cadd(x, cadd(y, cadd(d, e))); }
}

int main() {
  cplx* out; long long* cyc;
  cudaMalloc(&out, 16 * 4); cudaMalloc(&cyc, 8 * 4);
  const int steps = 10000;
  for (int rep = 0; rep < 2; ++rep) {
    front<0><<<1, 32>>>(out, cyc, steps, cmk(0.1, 0.2), cmk(0.9, 0.1), cmk(0.3, 0.3));
    front<1><<<1, 32>>>(out, cyc, steps, cmk(0.1, 0.2), cmk(0.9, 0.1), cmk(0.3, 0.3));
    front<2><<<1, 32>>>(out, cyc, steps, cmk(0.1, 0.2), cmk(0.9, 0.1), cmk(0.3, 0.3));
  }
  long long h[4];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("front step: rsqrt %.1f cyc, f32 seed+2N %.1f cyc, f32 seed+3N %.1f cyc\n", (double)h[0] / steps,
         (double)h[1] / steps, (double)h[2] / steps);
  return 0;
}
