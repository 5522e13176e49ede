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
  int splits = 1;                     // split-K slices (> 1: raw partial sums into part)
  cplx* part = nullptr;               // splits x batch x M x N partials
  const long long* a_ptrs = nullptr;  // optional: A of batch entry b at address a_ptrs[b] (sA ignored)
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
  const int b = blockIdx.z / g.splits, ks = blockIdx.z % g.splits;
  // k range of this slice (a multiple of GBK wide)
  const int kc = ((g.K + g.splits - 1) / g.splits + GBK - 1) / GBK * GBK;
  const int kbeg = ks * kc, kend = min(g.K, kbeg + kc);
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;  // warp tile origin
  const cplx* Bg = g.B + (long long)b * g.sB;
  cplx* Cg = g.C + (long long)b * g.sC;

  auto load_tile = [&](int stage, int k0) {
    unsigned char* base = gsm + stage * S::stage;
    if constexpr (A_REAL) {
      const double* Ag = g.a_ptrs ? reinterpret_cast<const double*>(g.a_ptrs[b])
                                  : reinterpret_cast<const double*>(g.A) + (long long)b * g.sA;
      double* As = reinterpret_cast<double*>(base);
#pragma unroll
      for (int i = 0; i < (GBM * GBK) / GTHREADS; ++i) {
        int e = tid + i * GTHREADS, r = e / GBK, c = e % GBK;
        int gr = m0 + r, gc = k0 + c;
        bool p = gr < g.M && gc < kend;
        const double* src = p ? Ag + (long long)gr * g.lda + gc : Ag;
        cp_async8(As + r * GAR_LD + c, src, p);
      }
    } else {
      const cplx* Ag = g.a_ptrs ? reinterpret_cast<const cplx*>(g.a_ptrs[b])
                                : reinterpret_cast<const cplx*>(g.A) + (long long)b * g.sA;
      cplx* As = reinterpret_cast<cplx*>(base);
#pragma unroll
      for (int i = 0; i < (GBM * GBK) / GTHREADS; ++i) {
        int e = tid + i * GTHREADS, r = e / GBK, c = e % GBK;
        int gr = m0 + r, gc = k0 + c;
        bool p = gr < g.M && gc < kend;
        const cplx* src = p ? Ag + (long long)gr * g.lda + gc : Ag;
        cp_async16(As + r * GA_LD + c, src, p);
      }
    }
    cplx* Bs = reinterpret_cast<cplx*>(base + S::a_bytes);
#pragma unroll
    for (int i = 0; i < (GBK * GBN) / GTHREADS; ++i) {
      int e = tid + i * GTHREADS, r = e / GBN, c = e % GBN;
      int gr = k0 + r, gc = n0 + c;
      bool p = gr < kend && gc < g.N;
      const cplx* src = p ? Bg + (long long)gr * g.ldb + gc : Bg;
      cp_async16(Bs + r * GB_LD + c, src, p);
    }
  };

  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

  const int ktiles = kend > kbeg ? (kend - kbeg + GBK - 1) / GBK : 0;
  if (ktiles > 0) load_tile(0, kbeg);
  cp_async_commit();
  for (int kt = 0; kt < ktiles; ++kt) {
    if (kt + 1 < ktiles) load_tile((kt + 1) & 1, kbeg + (kt + 1) * GBK);
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
        if (c + h < g.N && g.splits > 1) {
          g.part[((long long)(ks * g.batch + b) * g.M + r) * g.N + c + h] = cmk(cr[i][j][h], ci[i][j][h]);
        } else if (c + h < g.N) {
          cplx* dst = Cg + (long long)r * g.ldc + c + h;
          cplx v = cmk(g.alpha * cr[i][j][h], g.alpha * ci[i][j][h]);
          if (g.beta) v = cadd(*dst, v);
          *dst = v;
        }
      }
    }
  }
}

// C = beta C + alpha sum_s part[s] in fixed slice order (deterministic split-K)
static __global__ void splitk_reduce_kernel(GemmArgs g) {
  const long long mn = (long long)g.M * g.N;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= mn * g.batch) return;
  const int b = (int)(e / mn);
  const long long rc = e % mn;
  const int r = (int)(rc / g.N), c = (int)(rc % g.N);
  double sr = 0.0, si = 0.0;
  for (int s = 0; s < g.splits; ++s) {
    const cplx v = g.part[(long long)(s * g.batch + b) * mn + rc];
    sr += v.x;
    si += v.y;
  }
  cplx* dst = g.C + (long long)b * g.sC + (long long)r * g.ldc + c;
  cplx v = cmk(g.alpha * sr, g.alpha * si);
  if (g.beta) v = cadd(*dst, v);
  *dst = v;
}

// Launch helper (host).  Returns 0 or a cudaError_t.  When the output tiles
// cannot fill the GPU twice over and K is long (the Q^H (A Q) and Gram
// products: 118 x 118 outputs over K = 4096), K is split into slices whose
// partial sums go to a stream-ordered scratch buffer and are reduced in a
// fixed order.
template <bool A_REAL, bool A_CONJ>
inline int gemm_launch(const GemmArgs& g0, cudaStream_t stream) {
  if (g0.M <= 0 || g0.N <= 0 || g0.batch <= 0) return 0;
  using S = GemmSmem<A_REAL>;
  static bool attr_set = false;
  static int sms = 0;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_kernel<A_REAL, A_CONJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::total);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // keep the split-K scratch in the stream-ordered pool across synchronisations
    // (the default release threshold of 0 would hand it back to the OS every time)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      unsigned long long keep = 1ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    attr_set = true;
  }
  if (g0.K <= 0) return 0;  // callers handle beta with K == 0 themselves
  GemmArgs g = g0;
  const long long tiles = (long long)((g.N + GBN - 1) / GBN) * ((g.M + GBM - 1) / GBM) * g.batch;
  int splits = 1;
  if (tiles < 2LL * sms && g.K >= 8 * GBK) {
    splits = (int)((2LL * sms + tiles - 1) / tiles);
    splits = splits < g.K / (4 * GBK) ? splits : g.K / (4 * GBK);   // >= 4 k-tiles per slice
    splits = splits < 64 ? splits : 64;
  }
  cudaError_t e;
  if (splits > 1) {
    g.splits = splits;
    e = cirr_malloc_async(reinterpret_cast<void**>(&g.part), sizeof(cplx) * (size_t)splits * g.batch * g.M * g.N,
                          stream);
    if (e != cudaSuccess) return (int)e;
  }
  dim3 grid((g.N + GBN - 1) / GBN, (g.M + GBM - 1) / GBM, g.batch * g.splits);
  gemm_kernel<A_REAL, A_CONJ><<<grid, GTHREADS, S::total, stream>>>(g);
  cirr_note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  if (splits > 1) {
    const long long total = (long long)g.batch * g.M * g.N;
    splitk_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(g);
    cirr_note_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    e = cudaFreeAsync(g.part, stream);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

}  // namespace cirr
