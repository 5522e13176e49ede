// Batched complex128 GEMM on the FP64 tensor pipe (mma.sync m8n8k4 f64 ->
// SASS DMMA.8x8x4).  Row-major operands, complex interleaved in global and
// shared memory; each complex 8x8x4 step is four real DMMAs
// (Cr += ar br - ai bi, Ci += ar bi + ai br); a real A operand needs two.
//
//   C[b] = beta * C[b] + alpha * op(A[b]) * B[b]     (beta in {0, 1}, alpha real)
//   op(A) = A or conj(A) (elementwise; no transpose), A complex or real f64.
//
// Used for the LU trailing update (A22 -= L21 U12, K2), B*V / A*Q / B*Q /
// Q^H(AQ) (K5) and X = Q s, A X, B X (K7).  Tiles: 64x64 complex per CTA,
// BK = 16, 8 warps as 2x4 with 32x16 warp tiles, cp.async double buffering
// into padded shared memory (conflict-free 16-byte fragment loads).
#pragma once
#include "common.cuh"

namespace cirr {

struct GemmArgs {
  int M, N, K, batch;
  const void* A; long long lda, sA;   // sA = batch stride in elements (0 = shared)
  const cplx* B; long long ldb, sB;
  cplx* C; long long ldc, sC;
  double alpha; int beta;             // beta: 0 -> overwrite, 1 -> accumulate
};

constexpr int GBM = 64, GBN = 64, GBK = 16;
constexpr int GTHREADS = 256;
constexpr int GA_LD = GBK + 4;        // complex per A smem row (320 B)
constexpr int GAR_LD = GBK + 4;       // doubles per real-A smem row (160 B)
constexpr int GB_LD = GBN + 2;        // complex per B smem row (1056 B)

template <bool A_REAL>
struct GemmSmem {
  static constexpr int a_bytes = A_REAL ? GBM * GAR_LD * 8 : GBM * GA_LD * 16;
  static constexpr int b_bytes = GBK * GB_LD * 16;
  static constexpr int stage = a_bytes + b_bytes;
  static constexpr int total = 2 * stage;
};

template <bool A_REAL, bool A_CONJ>
__global__ void __launch_bounds__(GTHREADS, 2) gemm_kernel(GemmArgs g) {
  extern __shared__ __align__(16) unsigned char gsm[];
  using S = GemmSmem<A_REAL>;
  const int b = blockIdx.z;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;  // warp tile origin
  const cplx* Bg = g.B + (long long)b * g.sB;
  cplx* Cg = g.C + (long long)b * g.sC;

  auto load_tile = [&](int stage, int k0) {
    unsigned char* base = gsm + stage * S::stage;
    if constexpr (A_REAL) {
      const double* Ag = reinterpret_cast<const double*>(g.A) + (long long)b * g.sA;
      double* As = reinterpret_cast<double*>(base);
#pragma unroll
      for (int i = 0; i < (GBM * GBK) / GTHREADS; ++i) {
        int e = tid + i * GTHREADS, r = e / GBK, c = e % GBK;
        int gr = m0 + r, gc = k0 + c;
        bool p = gr < g.M && gc < g.K;
        const double* src = p ? Ag + (long long)gr * g.lda + gc : Ag;
        cp_async8(As + r * GAR_LD + c, src, p);
      }
    } else {
      const cplx* Ag = reinterpret_cast<const cplx*>(g.A) + (long long)b * g.sA;
      cplx* As = reinterpret_cast<cplx*>(base);
#pragma unroll
      for (int i = 0; i < (GBM * GBK) / GTHREADS; ++i) {
        int e = tid + i * GTHREADS, r = e / GBK, c = e % GBK;
        int gr = m0 + r, gc = k0 + c;
        bool p = gr < g.M && gc < g.K;
        const cplx* src = p ? Ag + (long long)gr * g.lda + gc : Ag;
        cp_async16(As + r * GA_LD + c, src, p);
      }
    }
    cplx* Bs = reinterpret_cast<cplx*>(base + S::a_bytes);
#pragma unroll
    for (int i = 0; i < (GBK * GBN) / GTHREADS; ++i) {
      int e = tid + i * GTHREADS, r = e / GBN, c = e % GBN;
      int gr = k0 + r, gc = n0 + c;
      bool p = gr < g.K && gc < g.N;
      const cplx* src = p ? Bg + (long long)gr * g.ldb + gc : Bg;
      cp_async16(Bs + r * GB_LD + c, src, p);
    }
  };

  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

  const int ktiles = (g.K + GBK - 1) / GBK;
  load_tile(0, 0);
  cp_async_commit();
  for (int kt = 0; kt < ktiles; ++kt) {
    if (kt + 1 < ktiles) load_tile((kt + 1) & 1, (kt + 1) * GBK);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    unsigned char* base = gsm + (kt & 1) * S::stage;
    const cplx* Bs = reinterpret_cast<const cplx*>(base + S::a_bytes);
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      cplx bf[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bs[(kk + (lane & 3)) * GB_LD + wn + j * 8 + (lane >> 2)];
      if constexpr (A_REAL) {
        const double* As = reinterpret_cast<const double*>(base);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double a = As[(wm + i * 8 + (lane >> 2)) * GAR_LD + kk + (lane & 3)];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            dmma884(cr[i][j][0], cr[i][j][1], a, bf[j].x);
            dmma884(ci[i][j][0], ci[i][j][1], a, bf[j].y);
          }
        }
      } else {
        const cplx* As = reinterpret_cast<const cplx*>(base);
        cplx af[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          af[i] = As[(wm + i * 8 + (lane >> 2)) * GA_LD + kk + (lane & 3)];
          if (A_CONJ) af[i].y = -af[i].y;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            dmma884(cr[i][j][0], cr[i][j][1], af[i].x, bf[j].x);
            dmma884(ci[i][j][0], ci[i][j][1], af[i].x, bf[j].y);
          }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            dmma884(cr[i][j][0], cr[i][j][1], -af[i].y, bf[j].y);
            dmma884(ci[i][j][0], ci[i][j][1], af[i].y, bf[j].x);
          }
      }
    }
    __syncthreads();
  }
  // epilogue: lane holds C[r][c], C[r][c+1] of each 8x8 block
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = m0 + wm + i * 8 + (lane >> 2);
    if (r >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      int c = n0 + wn + j * 8 + 2 * (lane & 3);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (c + h < g.N) {
          cplx* dst = Cg + (long long)r * g.ldc + c + h;
          cplx v = cmk(g.alpha * cr[i][j][h], g.alpha * ci[i][j][h]);
          if (g.beta) v = cadd(*dst, v);
          *dst = v;
        }
      }
    }
  }
}

// Launch helper (host).  Returns 0 or a cudaError_t.
template <bool A_REAL, bool A_CONJ>
inline int gemm_launch(const GemmArgs& g, cudaStream_t stream) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return 0;
  using S = GemmSmem<A_REAL>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_kernel<A_REAL, A_CONJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::total);
    attr_set = true;
  }
  if (g.K <= 0) return 0;  // callers handle beta with K == 0 themselves
  dim3 grid((g.N + GBN - 1) / GBN, (g.M + GBM - 1) / GBM, g.batch);
  gemm_kernel<A_REAL, A_CONJ><<<grid, GTHREADS, S::total, stream>>>(g);
  cirr_note_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // namespace cirr
