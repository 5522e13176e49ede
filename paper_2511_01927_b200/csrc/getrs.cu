// K3: batched multi-RHS triangular solves against the LU factors, plus the
// quadrature moment accumulation.
//
// Replaces linalg.py:46-52 (SuperLU gstrs) and solvers.py:113-130
// (ProjectorContext.apply: BV once, then per node Y_j = (z_j B - A)^-1 BV and
// S_m += w_j zeta_j^m Y_j).  Y_j = U^-1 L^-1 P BV_c(j):
//   * permute_kernel gathers the contour's RHS rows through perm_j;
//   * trsm_blocked_kernel<LOWER> walks 64-row blocks of one pencil for a
//     32-column RHS chunk: the off-diagonal contribution sum_l T_il Y_l is a
//     DMMA GEMM (cp.async double-buffered), the 64x64 diagonal block is
//     solved in shared memory;
//   * moments_kernel sums the nodes of each contour in fixed order
//     (deterministic, test_solvers.py:192-198) reading every Y_j once and
//     writes S transposed (one contiguous row per column of S) for K4.
#include "common.cuh"
#include <cstdlib>
#include "lu_gemm.cuh"
#include "ozaki.cuh"

namespace {

constexpr int SNB = 64;           // block rows
constexpr int SKC = 32;           // RHS columns per CTA (the wide variant)
constexpr int SBK = 16;           // GEMM k-step
constexpr int SA_LD = SBK + 4;    // complex per A smem row
constexpr int SD_LD = SNB + 1;    // diagonal block row
constexpr int kStageA = SNB * SA_LD;
// The left-looking kernel in two widths: KC = 32 RHS columns per CTA (256
// threads, 93 KB: two CTAs per SM) and KC = 16 for K <= 16 (128 threads,
// 68 KB: three CTAs per SM, half the padded DMMA work at config 2's K = 8..16).
// The diagonal block is kept packed (its triangle only, element (hi, lo) at
// hi (hi + 1) / 2 + lo) in the cp.async stage area, which is idle while the
// block is solved.
template <int KC>
struct SolveCfg {
  static constexpr int NT = 8 * KC;                 // threads
  static constexpr int B_LD = KC + 2;               // complex per B smem row
  static constexpr int X_LD = KC + 1;
  static constexpr int kStageB = SBK * B_LD;
  static constexpr int kSmem = (2 * (kStageA + kStageB) + SNB * X_LD + SNB) * 16;
};
constexpr int kPackedD = SNB * (SNB + 1) / 2;
static_assert(kPackedD <= 2 * (kStageA + SolveCfg<16>::kStageB), "packed diagonal block must fit the stage area");
__device__ __forceinline__ int pk_tri(int hi, int lo) { return hi * (hi + 1) / 2 + lo; }

template <bool LOWER, int KC>
__global__ void __launch_bounds__(8 * KC, KC == 32 ? 2 : 3) trsm_blocked_kernel(const cplx* __restrict__ LU, long long ld,
                                                              long long pstride, int n,
                                                              cplx* __restrict__ Y, long long ldy,
                                                              long long ystride, int K,
                                                              const int* __restrict__ pmap, int klL, int kuU) {
  using CF = SolveCfg<KC>;
  constexpr int NT = CF::NT, SB_LD = CF::B_LD, SX_LD = CF::X_LD, kStageB = CF::kStageB, SKC_ = KC;
  extern __shared__ __align__(16) cplx ssm[];
  cplx* stA = ssm;                                   // 2 stages
  cplx* stB = ssm + 2 * kStageA;
  cplx* D = ssm;                                     // packed diagonal block (aliases the stages)
  cplx* X = ssm + 2 * (kStageA + kStageB);           // RHS block
  cplx* dinv = X + SNB * SX_LD;
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * SKC_;
  const cplx* T = LU + (long long)(pmap ? pmap[b] : b) * pstride;
  cplx* Yb = Y + (long long)b * ystride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / (KC / 16)) * 16, wn = (warp % (KC / 16)) * 16;
  const int nblk = (n + SNB - 1) / SNB;

  for (int step = 0; step < nblk; ++step) {
    const int bi = LOWER ? step : nblk - 1 - step;
    const int i0 = bi * SNB;
    const int nbi = min(SNB, n - i0);
    // k-range of the off-diagonal product
    // off-diagonal range, cut to the band: L_ik = 0 for i - k > klL and
    // U_ik = 0 for k - i > kuU
    // (the lower start on the k-step grid of the full range, so every k-step
    // sums the same products as the dense solve: bitwise equal results)
    const int kbeg = LOWER ? max(0, i0 - (klL + SBK - 1) / SBK * SBK) : i0 + nbi;
    const int kend = LOWER ? i0 : min(n, i0 + nbi + kuU);
    const int klen = kend - kbeg;

    double cr[2][2][2], ci[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

    auto load = [&](int stage, int kk) {
      cplx* As = stA + stage * kStageA;
      cplx* Bs = stB + stage * kStageB;
#pragma unroll
      for (int t = 0; t < (SNB * SBK) / NT; ++t) {
        int e = tid + t * NT, r = e / SBK, c = e % SBK;
        int gr = i0 + r, gc = kbeg + kk + c;
        bool p = r < nbi && gc < kend;
        cp_async16(As + r * SA_LD + c, p ? T + (long long)gr * ld + gc : T, p);
      }
#pragma unroll
      for (int t = 0; t < (SBK * SKC_) / NT; ++t) {
        int e = tid + t * NT, r = e / SKC_, c = e % SKC_;
        int gr = kbeg + kk + r, gc = c0 + c;
        bool p = gr < kend && gc < K;
        cp_async16(Bs + r * SB_LD + c, p ? Yb + (long long)gr * ldy + gc : Yb, p);
      }
    };

    if (klen > 0) {
      const int kt = (klen + SBK - 1) / SBK;
      load(0, 0);
      cp_async_commit();
      for (int t = 0; t < kt; ++t) {
        if (t + 1 < kt) load((t + 1) & 1, (t + 1) * SBK);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const cplx* As = stA + (t & 1) * kStageA;
        const cplx* Bs = stB + (t & 1) * kStageB;
#pragma unroll
        for (int kk = 0; kk < SBK; kk += 4) {
          cplx af[2], bf[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) af[i] = As[(wm + i * 8 + (lane >> 2)) * SA_LD + kk + (lane & 3)];
#pragma unroll
          for (int j = 0; j < 2; ++j) bf[j] = Bs[(kk + (lane & 3)) * SB_LD + wn + j * 8 + (lane >> 2)];
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              dmma884(cr[i][j][0], cr[i][j][1], af[i].x, bf[j].x);
              dmma884(ci[i][j][0], ci[i][j][1], af[i].x, bf[j].y);
            }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              dmma884(cr[i][j][0], cr[i][j][1], -af[i].y, bf[j].y);
              dmma884(ci[i][j][0], ci[i][j][1], af[i].y, bf[j].x);
            }
        }
        __syncthreads();
      }
    }
    // load the diagonal block's triangle (packed) and the RHS block
    for (int e = tid; e < SNB * SNB; e += NT) {
      int r = e / SNB, c = e % SNB;
      if (LOWER ? c <= r : r <= c)
        D[LOWER ? pk_tri(r, c) : pk_tri(c, r)] =
            (r < nbi && c < nbi) ? T[(long long)(i0 + r) * ld + i0 + c] : cmk(0.0, 0.0);
    }
    for (int e = tid; e < SNB * SKC_; e += NT) {
      int r = e / SKC_, c = e % SKC_;
      X[r * SX_LD + c] = (r < nbi && c0 + c < K) ? Yb[(long long)(i0 + r) * ldy + c0 + c] : cmk(0.0, 0.0);
    }
    __syncthreads();
    // X -= accumulated off-diagonal product
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int r = wm + i * 8 + (lane >> 2), c = wn + j * 8 + 2 * (lane & 3) + h;
          cplx v = X[r * SX_LD + c];
          X[r * SX_LD + c] = cmk(v.x - cr[i][j][h], v.y - ci[i][j][h]);
        }
    if (!LOWER && tid < SNB) dinv[tid] = tid < nbi ? crecip(D[pk_tri(tid, tid)]) : cmk(0.0, 0.0);
    __syncthreads();
    // diagonal solve without CTA barriers: warp w owns columns 4w .. 4w+3,
    // lane l rows l and l + 32 in registers; each finished row is broadcast
    // by a shuffle (the first version ran one CTA barrier per row: 63 per
    // block, the latency chain of config 2's small solves)
    {
      const int cb = warp * 4;
      if (c0 + cb < K) {
        cplx xr[2][4];
#pragma unroll
        for (int sl = 0; sl < 2; ++sl)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) xr[sl][cc] = X[(lane + 32 * sl) * SX_LD + cb + cc];
        if (LOWER) {
          for (int i = 0; i < nbi - 1; ++i) {
            const int src = i & 31;
            const bool hi = i >= 32;
            cplx xi[4];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              const cplx v = hi ? xr[1][cc] : xr[0][cc];
              xi[cc] = cmk(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
            }
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
              const int r = lane + 32 * sl;
              if (r > i && r < nbi) {
                const cplx d = D[pk_tri(r, i)];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) cfms(xr[sl][cc], d, xi[cc]);
              }
            }
          }
        } else {
          for (int i = nbi - 1; i >= 0; --i) {
            const int src = i & 31;
            const bool hi = i >= 32;
            const cplx di = dinv[i];
            cplx xi[4];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              const cplx v = cmul(hi ? xr[1][cc] : xr[0][cc], di);
              xi[cc] = cmk(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
              if (lane == src) {
                if (hi) xr[1][cc] = xi[cc];
                else xr[0][cc] = xi[cc];
              }
            }
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
              const int r = lane + 32 * sl;
              if (r < i) {
                const cplx d = D[pk_tri(i, r)];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) cfms(xr[sl][cc], d, xi[cc]);
              }
            }
          }
        }
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          const int r = lane + 32 * sl;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            if (r < nbi && c0 + cb + cc < K) Yb[(long long)(i0 + r) * ldy + c0 + cb + cc] = xr[sl][cc];
        }
      }
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// 128 x 128 diagonal-block inverses for the right-looking solve: with DB = 128
// the trailing GEMMs run with k = 128 (half the launches and half the C-tile
// traffic of k = 64).  Each inverse is assembled from two 64 x 64 triangular
// inverses and one off-diagonal block:
//   lower  [[L11, 0], [L21, L22]]^-1 = [[X1, 0], [-X2 L21 X1, X2]]
//   upper  [[U11, U12], [0, U22]]^-1 = [[X1, -X1 U12 X2], [0, X2]]
constexpr int DB = 128;

// X = T^-1 for the nb x nb (nb <= 64) triangular block in D (smem, ld SD_LD);
// lower: unit diagonal; X is identity-padded outside nb.  256 threads: column
// j of X in four threads that split each dot product (two shuffles combine
// it), so the substitution needs no CTA barrier (the first version ran one
// barrier per row, 63 per inverse: config 4's diagonal inverses 8.3 ms).
template <bool LOWER>
__device__ void tri_inv64(const cplx* D, cplx* X, cplx* dinv, int nb) {
  const int tid = threadIdx.x;
  for (int e = tid; e < SNB * SNB; e += 256) {
    const int r = e / SNB, c = e % SNB;
    X[r * SD_LD + c] = cmk((r == c && r < nb) ? 1.0 : 0.0, 0.0);
  }
  if (!LOWER && tid < nb) dinv[tid] = crecip(D[tid * SD_LD + tid]);
  __syncthreads();
  const int j = tid >> 2, q = tid & 3;
  if (LOWER) {
    for (int i = 1; i < nb; ++i) {
      double sr = 0.0, si = 0.0;
      for (int kk = q; kk < i; kk += 4) {
        if (kk >= j) {
          const cplx a = D[i * SD_LD + kk], x = X[kk * SD_LD + j];
          sr = fma(a.x, x.x, sr); sr = fma(-a.y, x.y, sr);
          si = fma(a.x, x.y, si); si = fma(a.y, x.x, si);
        }
      }
      sr += __shfl_xor_sync(0xffffffffu, sr, 1); si += __shfl_xor_sync(0xffffffffu, si, 1);
      sr += __shfl_xor_sync(0xffffffffu, sr, 2); si += __shfl_xor_sync(0xffffffffu, si, 2);
      if (q == 0 && i > j) X[i * SD_LD + j] = cmk(-sr, -si);
      __syncwarp();
    }
  } else {
    for (int i = nb - 1; i >= 0; --i) {
      double sr = 0.0, si = 0.0;
      for (int kk = i + 1 + q; kk < nb; kk += 4) {
        if (kk <= j) {
          const cplx a = D[i * SD_LD + kk], x = X[kk * SD_LD + j];
          sr = fma(a.x, x.x, sr); sr = fma(-a.y, x.y, sr);
          si = fma(a.x, x.y, si); si = fma(a.y, x.x, si);
        }
      }
      sr += __shfl_xor_sync(0xffffffffu, sr, 1); si += __shfl_xor_sync(0xffffffffu, si, 1);
      sr += __shfl_xor_sync(0xffffffffu, sr, 2); si += __shfl_xor_sync(0xffffffffu, si, 2);
      if (q == 0 && i <= j && j < nb) X[i * SD_LD + j] = cmul(cmk((i == j ? 1.0 : 0.0) - sr, -si), dinv[i]);
      __syncwarp();
    }
  }
  __syncthreads();
}

// T <- sign * (L @ R) for 64 x 64 smem blocks (in place into T allowed when T
// aliases L or R: every product is held in registers before the write-back).
__device__ void mm64_inplace(const cplx* L, const cplx* R, cplx* T, double sign) {
  const int tid = threadIdx.x;
  cplx acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int e = tid + q * 256, r = e / SNB, c = e % SNB;
    cplx a = cmk(0.0, 0.0);
    for (int k = 0; k < SNB; ++k) cfma(a, L[r * SD_LD + k], R[k * SD_LD + c]);
    acc[q] = cmk(sign * a.x, sign * a.y);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int e = tid + q * 256;
    T[(e / SNB) * SD_LD + e % SNB] = acc[q];
  }
  __syncthreads();
}

template <bool LOWER>
__global__ void __launch_bounds__(256) diag_inv128_kernel(const cplx* __restrict__ LU, long long ld,
                                                          long long pstride, int n, cplx* __restrict__ Dinv) {
  extern __shared__ __align__(16) cplx ism[];
  cplx* X1 = ism;
  cplx* X2 = X1 + SNB * SD_LD;
  cplx* T = X2 + SNB * SD_LD;
  cplx* dinv = T + SNB * SD_LD;
  const int bi = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int nblk = gridDim.x;
  const int i0 = bi * DB, nb = min(DB, n - i0);
  const int na = min(SNB, nb), nb2 = nb - na;
  const cplx* A = LU + (long long)b * pstride;
  auto load = [&](cplx* dst, int r0, int c0, int nr, int nc) {
    for (int e = tid; e < SNB * SNB; e += 256) {
      const int r = e / SNB, c = e % SNB;
      dst[r * SD_LD + c] = (r < nr && c < nc) ? A[(long long)(r0 + r) * ld + c0 + c] : cmk(0.0, 0.0);
    }
    __syncthreads();
  };
  load(T, i0, i0, na, na);
  tri_inv64<LOWER>(T, X1, dinv, na);
  if (nb2 > 0) {
    load(T, i0 + SNB, i0 + SNB, nb2, nb2);
    tri_inv64<LOWER>(T, X2, dinv, nb2);
    if (LOWER) {
      load(T, i0 + SNB, i0, nb2, na);       // L21
      mm64_inplace(T, X1, T, 1.0);          // L21 X1
      mm64_inplace(X2, T, T, -1.0);         // -X2 L21 X1
    } else {
      load(T, i0, i0 + SNB, na, nb2);       // U12
      mm64_inplace(T, X2, T, 1.0);          // U12 X2
      mm64_inplace(X1, T, T, -1.0);         // -X1 U12 X2
    }
  }
  cplx* out = Dinv + (((long long)b * nblk + bi) * 2 + (LOWER ? 0 : 1)) * DB * DB;
  for (int e = tid; e < DB * DB; e += 256) {
    const int r = e / DB, c = e % DB;
    const bool top = r < SNB, left = c < SNB;
    cplx v = cmk(0.0, 0.0);
    if (top && left) v = X1[r * SD_LD + c];
    else if (!top && !left) v = nb2 > 0 ? X2[(r - SNB) * SD_LD + c - SNB] : cmk(0.0, 0.0);
    else if (LOWER && !top && left) v = nb2 > 0 ? T[(r - SNB) * SD_LD + c] : cmk(0.0, 0.0);
    else if (!LOWER && top && !left) v = nb2 > 0 ? T[r * SD_LD + c - SNB] : cmk(0.0, 0.0);
    out[e] = v;
  }
}
constexpr int kDiagInv128Smem = (3 * SNB * SD_LD + SNB) * 16;

// Y[j][i][c] = R[rhs_of[j]][perm[j][i]][c]
__global__ void permute_kernel(const cplx* __restrict__ R, long long ldr, long long rstride,
                               const int* __restrict__ rhs_of, const int* __restrict__ perm, int n, int K,
                               cplx* __restrict__ Y, long long ldy, long long ystride,
                               const int* __restrict__ pmap) {
  const int j = blockIdx.y;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * K) return;
  const int i = (int)(e / K), c = (int)(e % K);
  const cplx* Rj = R + (long long)rhs_of[j] * rstride;
  const int src = perm[(long long)(pmap ? pmap[j] : j) * n + i];
  Y[(long long)j * ystride + (long long)i * ldy + c] = Rj[(long long)src * ldr + c];
}

constexpr int MAXM = 16;
constexpr int MTR = 32;       // rows per tile
constexpr int MTC = 32;       // columns per tile
// St[c][m*K + col][r] = sum_{j in contour c, in order} coef[j][m] * Y_j[r][col].
// One CTA per (32-row x 32-column tile, contour): every node's tile is read as
// 32 contiguous 512-byte row segments, the sums stay in registers (4 elements
// per thread), and S^T is written back through a shared-memory transpose so
// its rows (contiguous along r) are also written in 512-byte runs.  HBM-bound:
// each Y_j is read exactly once.
template <int MM, int RQ>
__global__ void __launch_bounds__(256) moments_kernel(const cplx* __restrict__ Y, long long ldy,
                                                      long long ystride, int n, int K,
                                                      const cplx* __restrict__ coef, int M,
                                                      const int* __restrict__ off, cplx* __restrict__ St,
                                                      long long ld_st, long long sstride, int row_lo) {
  constexpr int TR = 8 * RQ;  // rows per tile: 32 for whole-matrix calls, 8 for the 128-row windows of a solve
  __shared__ cplx tile[MTC][TR + 1];
  const int cidx = blockIdx.z;
  const int r0 = row_lo + blockIdx.y * TR, c0 = blockIdx.x * MTC;
  const int tid = threadIdx.x;
  const int j0 = off[cidx], j1 = off[cidx + 1];
  const int nj = j1 - j0;
  const cplx* cj = coef + (long long)j0 * M;   // broadcast loads (same address in a warp)
  // element q of this thread: row r0 + (tid >> 5) + 8 q, column c0 + (tid & 31)
  const int cl = tid & 31, rl = tid >> 5;
  const int col = c0 + cl;
  cplx acc[RQ][MM];
#pragma unroll
  for (int q = 0; q < RQ; ++q)
#pragma unroll
    for (int m = 0; m < MM; ++m) acc[q][m] = cmk(0.0, 0.0);
  bool ok[RQ];
  long long base[RQ];
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    const int r = r0 + rl + 8 * q;
    ok[q] = r < n && col < K;
    base[q] = (long long)r * ldy + col;
  }
  const cplx* Yc = Y + (long long)j0 * ystride;
  for (int j = 0; j < nj; ++j, Yc += ystride) {
    cplx y[RQ];
#pragma unroll
    for (int q = 0; q < RQ; ++q) y[q] = ok[q] ? Yc[base[q]] : cmk(0.0, 0.0);
#pragma unroll
    for (int m = 0; m < MM; ++m)
      if (m < M) {
        const cplx cf = cj[j * M + m];
#pragma unroll
        for (int q = 0; q < RQ; ++q) cfma(acc[q][m], cf, y[q]);
      }
  }
  cplx* S = St + (long long)cidx * sstride;
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    if (m >= M) break;
#pragma unroll
    for (int q = 0; q < RQ; ++q) tile[cl][rl + 8 * q] = acc[q][m];
    __syncthreads();
    // write rows m*K + col of S^T: thread (rl', cl') writes S^T[c0 + rl' + 8q][r0 + cl']
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      const int e = tid + 256 * q, ce = e / TR, re = e % TR;
      const int cc = c0 + ce, rr = r0 + re;
      if (cc < K && rr < n) S[(long long)(m * K + cc) * ld_st + rr] = tile[ce][re];
    }
    __syncthreads();
  }
}

// Right-looking solve, diagonal step: Y[i0:i0+nb, c0:c0+64] <- T_ii^{-1} Y[...]
// (unit lower when LOWER, else upper with its diagonal), one CTA per
// (64-column chunk, pencil).
constexpr int DSC = 64;
constexpr int kDiagSmem = (SNB * SD_LD + SNB * (DSC + 1) + SNB) * 16;

template <bool LOWER>
__global__ void __launch_bounds__(256) diag_solve_kernel(const cplx* __restrict__ LU, long long ld, long long pstride,
                                                         int i0, int nb, cplx* __restrict__ Y, long long ldy,
                                                         long long ystride, int K, const int* __restrict__ pmap) {
  extern __shared__ __align__(16) cplx dsm[];
  cplx* D = dsm;
  cplx* X = D + SNB * SD_LD;
  cplx* dinv = X + SNB * (DSC + 1);
  const int b = blockIdx.y, c0 = blockIdx.x * DSC, tid = threadIdx.x;
  const cplx* T = LU + (long long)(pmap ? pmap[b] : b) * pstride;
  cplx* Yb = Y + (long long)b * ystride;
  const int nc = min(DSC, K - c0);
  for (int e = tid; e < nb * nb; e += 256) {
    const int r = e / nb, c = e % nb;
    D[r * SD_LD + c] = T[(long long)(i0 + r) * ld + i0 + c];
  }
  for (int e = tid; e < nb * DSC; e += 256) {
    const int r = e / DSC, c = e % DSC;
    X[r * (DSC + 1) + c] = c < nc ? Yb[(long long)(i0 + r) * ldy + c0 + c] : cmk(0.0, 0.0);
  }
  __syncthreads();
  if (!LOWER && tid < nb) dinv[tid] = crecip(D[tid * SD_LD + tid]);
  __syncthreads();
  const int c = tid % DSC, g = tid / DSC;  // 4 row groups
  if (LOWER) {
    for (int i = 0; i < nb - 1; ++i) {
      const cplx xi = X[i * (DSC + 1) + c];
      for (int r = i + 1 + g; r < nb; r += 4) cfms(X[r * (DSC + 1) + c], D[r * SD_LD + i], xi);
      __syncthreads();
    }
  } else {
    for (int i = nb - 1; i >= 0; --i) {
      const cplx xi = cmul(X[i * (DSC + 1) + c], dinv[i]);
      __syncthreads();
      if (g == 0) X[i * (DSC + 1) + c] = xi;
      for (int r = g; r < i; r += 4) cfms(X[r * (DSC + 1) + c], D[r * SD_LD + i], xi);
      __syncthreads();
    }
  }
  for (int e = tid; e < nb * DSC; e += 256) {
    const int r = e / DSC, cc = e % DSC;
    if (cc < nc) Yb[(long long)(i0 + r) * ldy + c0 + cc] = X[r * (DSC + 1) + cc];
  }
}

// Narrow right-hand sides (K <= 2, e.g. the Krylov scouts' single vector):
// decoupled look-back triangular solve.  One CTA per 128-row block of one
// pencil: it accumulates -T_ik y_k for the blocks k it depends on as soon as
// each y_k is published (flag per block, written after a release fence), then
// applies the precomputed inverse of its diagonal block and publishes y_i.
// Dependencies only point to lower CTA indices (the backward solve walks the
// blocks in reverse index order), so the launch order guarantees progress.
// Every tile is read once, coalesced (a warp reads 32 consecutive columns of
// 16 rows), and the chain costs one tile GEMV plus one handoff per block.
constexpr int TV_BS = 128;       // block rows (= the diagonal-inverse block DB)
constexpr int TV_T = 256;
template <int KK, bool LOWER>
__global__ void __launch_bounds__(TV_T) trsv_lookback_kernel(const cplx* __restrict__ LU, long long ld,
                                                             long long pstride, int n, const cplx* __restrict__ Dinv,
                                                             cplx* __restrict__ Y, long long ldy, long long ystride,
                                                             int* __restrict__ flags, const int* __restrict__ pmap) {
  __shared__ cplx sacc[TV_BS][KK];
  __shared__ cplx sy[TV_BS][KK];
  const int nblk = gridDim.x, b = blockIdx.y;
  const int bi = LOWER ? blockIdx.x : nblk - 1 - blockIdx.x;
  const int i0 = bi * TV_BS, nb = min(TV_BS, n - i0);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int pb = pmap ? pmap[b] : b;
  const cplx* T = LU + (long long)pb * pstride;
  cplx* Yb = Y + (long long)b * ystride;
  int* fl = flags + (long long)b * nblk;
  // warp wid owns rows i0 + 16 wid .. +15; lane covers columns c0 + lane (+32, +64, +96)
  cplx part[16][KK];
#pragma unroll
  for (int q = 0; q < 16; ++q)
#pragma unroll
    for (int c = 0; c < KK; ++c) part[q][c] = cmk(0.0, 0.0);
  auto tile = [&](const cplx* Tt, long long ldt, int ncols, const cplx (*yv)[KK], int nrows_here) {
    // part[q] += Tt[row q][col] * yv[col] over this lane's columns
#pragma unroll
    for (int cc = 0; cc < TV_BS; cc += 32) {
      const int col = cc + lane;
      cplx yc[KK];
#pragma unroll
      for (int c = 0; c < KK; ++c) yc[c] = col < ncols ? yv[col][c] : cmk(0.0, 0.0);
      cplx t[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int r = wid * 16 + q;
        t[q] = (r < nrows_here && col < ncols) ? Tt[(long long)r * ldt + col] : cmk(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q)
#pragma unroll
        for (int c = 0; c < KK; ++c) cfma(part[q][c], t[q], yc[c]);
    }
  };
  // dependencies in the order they are published: forward 0, 1, ..; backward nblk-1, nblk-2, ..
  const int ndep = LOWER ? bi : nblk - 1 - bi;
  for (int t = 0; t < ndep; ++t) {
    const int kb = LOWER ? t : nblk - 1 - t;
    const int k0 = kb * TV_BS, nk = min(TV_BS, n - k0);
    if (tid == 0) {
      while (*((volatile int*)(fl + kb)) == 0) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
    for (int e = tid; e < TV_BS * KK; e += TV_T) {
      const int r = e / KK, c = e % KK;
      sy[r][c] = r < nk ? Yb[(long long)(k0 + r) * ldy + c] : cmk(0.0, 0.0);
    }
    __syncthreads();
    tile(T + (long long)i0 * ld + k0, ld, nk, sy, nb);
    __syncthreads();
  }
  // acc = rhs - sum (lane partials reduced per row)
#pragma unroll
  for (int q = 0; q < 16; ++q)
#pragma unroll
    for (int c = 0; c < KK; ++c) {
      const double re = warp_sum(part[q][c].x), im = warp_sum(part[q][c].y);
      const int r = wid * 16 + q;
      if (lane == 0) sacc[r][c] = r < nb ? csub(Yb[(long long)(i0 + r) * ldy + c], cmk(re, im)) : cmk(0.0, 0.0);
    }
  __syncthreads();
  // y_i = Dinv_i acc
#pragma unroll
  for (int q = 0; q < 16; ++q)
#pragma unroll
    for (int c = 0; c < KK; ++c) part[q][c] = cmk(0.0, 0.0);
  const cplx* D = Dinv + (((long long)pb * nblk + bi) * 2 + (LOWER ? 0 : 1)) * TV_BS * TV_BS;
  tile(D, TV_BS, nb, sacc, nb);
#pragma unroll
  for (int q = 0; q < 16; ++q)
#pragma unroll
    for (int c = 0; c < KK; ++c) {
      const double re = warp_sum(part[q][c].x), im = warp_sum(part[q][c].y);
      const int r = wid * 16 + q;
      if (lane == 0 && r < nb) Yb[(long long)(i0 + r) * ldy + c] = cmk(re, im);
    }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    *((volatile int*)(fl + bi)) = 1;
  }
}

template <int KK>
int trsv_lookback(const cplx* LU, int n, long long ld, long long pstride, int batch, const cplx* Dinv, cplx* Y,
                  long long ldy, long long ystride, cudaStream_t stream, const int* pmap) {
  const int nblk = (n + TV_BS - 1) / TV_BS;
  int* flags = nullptr;
  cudaError_t e = cirr_malloc_async(reinterpret_cast<void**>(&flags), sizeof(int) * 2 * (size_t)nblk * batch, stream);
  if (e != cudaSuccess) return (int)e;
  if ((e = cudaMemsetAsync(flags, 0, sizeof(int) * 2 * (size_t)nblk * batch, stream)) != cudaSuccess) return (int)e;
  dim3 g(nblk, batch);
  trsv_lookback_kernel<KK, true><<<g, TV_T, 0, stream>>>(LU, ld, pstride, n, Dinv, Y, ldy, ystride, flags, pmap);
  CIRR_CHECK_LAUNCH();
  trsv_lookback_kernel<KK, false><<<g, TV_T, 0, stream>>>(LU, ld, pstride, n, Dinv, Y, ldy, ystride,
                                                          flags + (long long)nblk * batch, pmap);
  CIRR_CHECK_LAUNCH();
  return (int)cudaFreeAsync(flags, stream);
}

}  // namespace

// Y_j = (P_j^T L_j U_j)^{-1} R_{rhs_of[j]} for j < batch.  LU/perm from
// cirr_zgetrf_batched; R: (n_rhs_sets) x n x K, row-major, ld ldr, stride
// rstride; Y: batch x n x K (ld ldy, stride ystride).  rhs_of is a device
// int32 array.
// Bytes of the diagonal-block inverses cirr_diag_inverses writes.
CIRR_API long long cirr_diag_inv_bytes(int n, int batch) {
  const long long nblk = (n + DB - 1) / DB;
  return (long long)batch * nblk * 2 * DB * DB * 16;
}

// Inverses of the 128x128 diagonal blocks of every factor (once per factorisation,
// reused by every solve pass).
CIRR_API int cirr_diag_inverses(const cplx* LU, int n, long long ld, long long pencil_stride, int batch, cplx* Dinv,
                                cudaStream_t stream) {
  if (n <= 0 || batch <= 0) return CIRR_EINVAL;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(diag_inv128_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDiagInv128Smem);
    cudaFuncSetAttribute(diag_inv128_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDiagInv128Smem);
    attr = true;
  }
  dim3 g((n + DB - 1) / DB, batch);
  diag_inv128_kernel<true><<<g, 256, kDiagInv128Smem, stream>>>(LU, ld, pencil_stride, n, Dinv);
  CIRR_CHECK_LAUNCH();
  diag_inv128_kernel<false><<<g, 256, kDiagInv128Smem, stream>>>(LU, ld, pencil_stride, n, Dinv);
  CIRR_CHECK_LAUNCH();
  return 0;
}

// The right-looking TMA path serves K > 16; for small factors (n <= 512,
// CIRR_SOLVE_SMALL_N) the left-looking kernel keeps up to K = 32 (one 32-column
// chunk per pencil), so those solves need no diagonal-block inverses.
static bool solve_tma_path(int n, int K) {
  static const int small_n = getenv("CIRR_SOLVE_SMALL_N") ? atoi(getenv("CIRR_SOLVE_SMALL_N")) : 512;
  return K > 16 && n >= 64 && !(n <= small_n && K <= SKC);
}

// Whether cirr_zgetrs_batched reads Dinv for an n x K solve: the look-back
// TRSV (K <= 2) and the TMA blocked path do; the left-looking kernel does not,
// so callers can skip cirr_diag_inverses there.
CIRR_API int cirr_zgetrs_uses_dinv(int n, int K) { return K <= 2 || solve_tma_path(n, K); }

// Moment accumulation fused into a solve call (solvers.py:121-129): St[c] +=
// coef[j*M+m] Y_j over the batch entries off[c]..off[c+1]-1 of contour c.
struct MomentSpec {
  const cplx* coef;
  int M;
  const int* off;
  int n_sets;
  cplx* St;
  long long ld_st, sstride;
};
static int launch_moments(const cplx* Y, long long ldy, long long ystride, int n, int K, const cplx* coef, int M,
                          const int* off, int n_sets, cplx* St, long long ld_st, long long sstride, int row_lo,
                          int row_hi, cudaStream_t stream);
static int moments_rows(const MomentSpec* ms, const cplx* Y, long long ldy, long long ystride, int n, int K,
                        int row_lo, int row_hi, cudaStream_t stream) {
  if (ms == nullptr) return 0;
  return launch_moments(Y, ldy, ystride, n, K, ms->coef, ms->M, ms->off, ms->n_sets, ms->St, ms->ld_st,
                        ms->sstride, row_lo, row_hi, stream);
}

// Solves for batch entries j = 0..batch-1 against factor pmap[j] (pmap null:
// factor j) of the nfac factors at LU (pencil_stride apart); perm and Dinv are
// indexed by factor, R by rhs_of[j], Y by j.
static int getrs_impl(const cplx* LU, int n, long long ld, long long pencil_stride, int batch, int nfac,
                      const int* pmap, const int* perm, const cplx* R, long long ldr, long long rstride,
                      const int* rhs_of, int K, cplx* Y, long long ldy, long long ystride, const cplx* Dinv,
                      cudaStream_t stream, const MomentSpec* ms = nullptr, int klL = -1, int kuU = -1) {
  if (n <= 0 || batch <= 0 || nfac <= 0 || K < 0 || ldy < K || ldr < K) return CIRR_EINVAL;
  // factor bandwidths (L below, U above the diagonal); -1 = dense.  Every
  // product below is cut to the rows / k-range the band allows: the skipped
  // blocks are exact zeros, so the results are bitwise those of the full solve.
  klL = (klL < 0 || klL > n - 1) ? n - 1 : klL;
  kuU = (kuU < 0 || kuU > n - 1) ? n - 1 : kuU;
  auto up16 = [](int x) { return (x + 15) / 16 * 16; };
  if (ms != nullptr && (ms->M < 1 || ms->M > MAXM || ms->n_sets <= 0)) return CIRR_EINVAL;
  if (K == 0) return 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(trsm_blocked_kernel<true, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SolveCfg<32>::kSmem);
    cudaFuncSetAttribute(trsm_blocked_kernel<false, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SolveCfg<32>::kSmem);
    cudaFuncSetAttribute(trsm_blocked_kernel<true, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SolveCfg<16>::kSmem);
    cudaFuncSetAttribute(trsm_blocked_kernel<false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SolveCfg<16>::kSmem);
    attr = true;
  }
  dim3 gp((unsigned)(((long long)n * K + 255) / 256), batch);
  permute_kernel<<<gp, 256, 0, stream>>>(R, ldr, rstride, rhs_of, perm, n, K, Y, ldy, ystride, pmap);
  CIRR_CHECK_LAUNCH();
  if (Dinv != nullptr && K <= 2) {  // one or two RHS: look-back triangular solves
    if (K == 1) CIRR_TRY(trsv_lookback<1>(LU, n, ld, pencil_stride, batch, Dinv, Y, ldy, ystride, stream, pmap));
    else CIRR_TRY(trsv_lookback<2>(LU, n, ld, pencil_stride, batch, Dinv, Y, ldy, ystride, stream, pmap));
    return moments_rows(ms, Y, ldy, ystride, n, K, 0, n, stream);
  }
  // right-looking blocked solves: per 64-row block a diagonal solve, then the
  // rank-64 update of the remaining rows on the TMA/DMMA GEMM (zgemm_sub_tma)
  // narrow RHS blocks (K <= 16) stay on the left-looking kernel: the 64-wide
  // GEMM tile of the right-looking path would be mostly padding there (at K = 32
  // the TMA path is still faster: 18.7 ms vs 24.3 ms for 64 pencils, n = 4096)
  cirr::OperandMaps mT, mY;
  static const int bn_env = getenv("CIRR_SOLVE_BN") ? atoi(getenv("CIRR_SOLVE_BN")) : 0;
  // swizzled B boxes for the right-hand sides (CIRR_SOLVE_BSWZ=0: one plain box per stage)
  static const bool kBswz = getenv("CIRR_SOLVE_BSWZ") ? atoi(getenv("CIRR_SOLVE_BSWZ")) != 0 : true;
  const int BN = bn_env > 0 ? bn_env : cirr::pick_tile_n(K, kBswz);
  bool tma = solve_tma_path(n, K) && cirr::encode_a_map(&mT.a, LU, n, n, nfac, ld, pencil_stride) == 0 &&
             (kBswz ? cirr::encode_b_swz_map(&mY.b, Y, K, n, batch, ldy, ystride)
                    : cirr::encode_c128_map(&mY.b, Y, K, n, batch, ldy, ystride, BN, cirr::PBK)) == 0 &&
             cirr::encode_c128_map(&mY.c, Y, K, n, batch, ldy, ystride, BN, cirr::PBM) == 0;
  if (tma) {
    static bool dattr = false;
    if (!dattr) {
      cudaFuncSetAttribute(diag_solve_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDiagSmem);
      cudaFuncSetAttribute(diag_solve_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDiagSmem);
      dattr = true;
    }
    CUtensorMap mD;
    const int nblk2 = (n + DB - 1) / DB;
    const bool use_dinv = Dinv != nullptr &&
                          cirr::encode_a_map(&mD, Dinv, DB, DB, nfac * nblk2 * 2, DB, (long long)DB * DB) == 0;
    if (use_dinv) {
      // 128-row blocks grouped into super-blocks of SBK blocks.  Inside a
      // super-block the blocks are left-looking (block j first receives the
      // contributions of blocks 0..j-1 of the super-block, one GEMM), and each
      // diagonal block is applied as two in-place GEMMs (M = 64 each, so every
      // output tile reads only its own rows plus rows that GEMM does not
      // write); the rows below/above then get one trailing update with
      // k = 128 * SBK (fewer C-tile round trips per flop than k = 128).
      static const int sbk_env = getenv("CIRR_SOLVE_SBK") ? atoi(getenv("CIRR_SOLVE_SBK")) : 0;
      const int SBK = sbk_env > 0 ? sbk_env : (n >= 2048 ? 4 : (n >= 512 ? 2 : 1));
      auto apply_dinv = [&](int bi, bool lower) -> int {
        const int i0 = bi * DB, nb = min(DB, n - i0), na = min(SNB, nb), nb2 = nb - na;
        const int slot = bi * 2 + (lower ? 0 : 1);
        if (lower) {
          if (nb2 > 0)  // rows i0+64.. : [L21inv L22inv] [Y_a; Y_b]
            CIRR_TRY(cirr::zgemm_sub_maps(mD, mY.b, mY.c, nb2, K, nb, batch, SNB, 0, i0, 0, i0 + SNB, 0, Y, ldy,
                                          ystride, stream, /*beta=*/0, nblk2 * 2, slot, pmap, BN, kBswz));
          CIRR_TRY(cirr::zgemm_sub_maps(mD, mY.b, mY.c, na, K, na, batch, 0, 0, i0, 0, i0, 0, Y, ldy, ystride, stream,
                                        /*beta=*/0, nblk2 * 2, slot, pmap, BN, kBswz));
        } else {
          // rows i0.. : [U11inv U12inv] [Y_a; Y_b] first (reads the old Y_b), then Y_b
          CIRR_TRY(cirr::zgemm_sub_maps(mD, mY.b, mY.c, na, K, nb, batch, 0, 0, i0, 0, i0, 0, Y, ldy, ystride, stream,
                                        /*beta=*/0, nblk2 * 2, slot, pmap, BN, kBswz));
          if (nb2 > 0)
            CIRR_TRY(cirr::zgemm_sub_maps(mD, mY.b, mY.c, nb2, K, nb2, batch, SNB, SNB, i0 + SNB, 0, i0 + SNB, 0, Y,
                                          ldy, ystride, stream, /*beta=*/0, nblk2 * 2, slot, pmap, BN, kBswz));
        }
        return 0;
      };
      for (int sb0 = 0; sb0 < nblk2; sb0 += SBK) {  // forward: L (unit lower)
        const int sb1 = min(nblk2, sb0 + SBK);
        const int s0 = sb0 * DB, s1 = min(n, sb1 * DB);
        for (int bi = sb0; bi < sb1; ++bi) {
          const int i0 = bi * DB, nb = min(DB, n - i0);
          if (bi > sb0) {  // Y[i0:i0+nb] -= L[i0:i0+nb, kb:i0] Y[kb:i0], kb >= s0 cut to the band
            const int kb = max(s0, i0 - up16(min(i0 - s0, klL)));
            CIRR_TRY(cirr::zgemm_sub_maps(mT.a, mY.b, mY.c, nb, K, i0 - kb, batch, i0, kb, kb, 0, i0, 0, Y, ldy,
                                          ystride, stream, 1, 1, 0, pmap, BN, kBswz));
          }
          CIRR_TRY(apply_dinv(bi, true));
        }
        if (n - s1 > 0) {  // Y[s1:s1+m] -= L[s1:s1+m, kb:s1] Y[kb:s1] (m = klL rows below can be nonzero)
          const int kb = max(s0, s1 - up16(min(s1 - s0, klL)));
          // int8 tensor cores on the factor slices kept after the factorisation (ozaki.cu), else DMMA
          int orc = -1;
          if (klL >= n - 1)
            orc = cirr::ozaki_cached_update(LU, n, kb, s1 - kb, s1, n - s1, Y + (long long)kb * ldy, ldy, ystride,
                                            Y + (long long)s1 * ldy, ldy, ystride, K, batch, pmap, stream);
          if (orc > 0) return orc;
          if (orc < 0)
            CIRR_TRY(cirr::zgemm_sub_maps(mT.a, mY.b, mY.c, min(n - s1, klL), K, s1 - kb, batch, s1, kb, kb, 0, s1, 0,
                                          Y, ldy, ystride, stream, 1, 1, 0, pmap, BN, kBswz));
        }
      }
      const int nsb = (nblk2 + SBK - 1) / SBK;
      for (int sb = nsb - 1; sb >= 0; --sb) {  // backward: U
        const int sb0 = sb * SBK, sb1 = min(nblk2, sb0 + SBK);
        const int s0 = sb0 * DB, s1 = min(n, sb1 * DB);
        for (int bi = sb1 - 1; bi >= sb0; --bi) {
          const int i0 = bi * DB, nb = min(DB, n - i0);
          if (bi < sb1 - 1) {  // Y[i0:i0+nb] -= U[i0:i0+nb, i0+nb:ke] Y[i0+nb:ke], ke <= s1 cut to the band
            const int ke = min(s1, i0 + nb + up16(min(s1 - i0 - nb, kuU)));
            if (ke > i0 + nb)
              CIRR_TRY(cirr::zgemm_sub_maps(mT.a, mY.b, mY.c, nb, K, ke - i0 - nb, batch, i0, i0 + nb, i0 + nb, 0, i0,
                                            0, Y, ldy, ystride, stream, 1, 1, 0, pmap, BN, kBswz));
          }
          CIRR_TRY(apply_dinv(bi, false));
          // rows i0.. are final for every entry: their moment rows now, while
          // the block (batch x 128 x K) is still in L2
          CIRR_TRY(moments_rows(ms, Y, ldy, ystride, n, K, i0, i0 + nb, stream));
        }
        if (s0 > 0) {  // Y[r0:s0] -= U[r0:s0, s0:ke] Y[s0:ke] (rows within kuU above, their columns)
          const int r0 = max(0, s0 - kuU), ke = min(s1, s0 + up16(min(s1 - s0, kuU)));
          int orc = -1;
          if (kuU >= n - 1)
            orc = cirr::ozaki_cached_update(LU, n, s0, ke - s0, 0, s0, Y + (long long)s0 * ldy, ldy, ystride, Y, ldy,
                                            ystride, K, batch, pmap, stream);
          if (orc > 0) return orc;
          if (orc < 0)
            CIRR_TRY(cirr::zgemm_sub_maps(mT.a, mY.b, mY.c, s0 - r0, K, ke - s0, batch, r0, s0, s0, 0, r0, 0, Y, ldy,
                                          ystride, stream, 1, 1, 0, pmap, BN, kBswz));
        }
      }
      return 0;
    }
    const int nblk = (n + SNB - 1) / SNB;
    dim3 gd((K + DSC - 1) / DSC, batch);
    for (int bi = 0; bi < nblk; ++bi) {  // forward: L (unit lower)
      const int i0 = bi * SNB, nb = min(SNB, n - i0);
      diag_solve_kernel<true><<<gd, 256, kDiagSmem, stream>>>(LU, ld, pencil_stride, i0, nb, Y, ldy, ystride, K, pmap);
      CIRR_CHECK_LAUNCH();
      CIRR_TRY(cirr::zgemm_sub_maps(mT.a, mY.b, mY.c, min(n - i0 - nb, klL), K, nb, batch, i0 + nb, i0, i0, 0,
                                    i0 + nb, 0, Y, ldy, ystride, stream, 1, 1, 0, pmap, BN, kBswz));
    }
    for (int bi = nblk - 1; bi >= 0; --bi) {  // backward: U
      const int i0 = bi * SNB, nb = min(SNB, n - i0);
      diag_solve_kernel<false><<<gd, 256, kDiagSmem, stream>>>(LU, ld, pencil_stride, i0, nb, Y, ldy, ystride, K, pmap);
      CIRR_CHECK_LAUNCH();
      const int r0 = max(0, i0 - kuU);
      CIRR_TRY(cirr::zgemm_sub_maps(mT.a, mY.b, mY.c, i0 - r0, K, nb, batch, r0, i0, i0, 0, r0, 0, Y, ldy, ystride,
                                    stream, 1, 1, 0, pmap, BN, kBswz));
    }
    return moments_rows(ms, Y, ldy, ystride, n, K, 0, n, stream);
  }
  static const int kc_env = getenv("CIRR_SOLVE_KC") ? atoi(getenv("CIRR_SOLVE_KC")) : 0;
  if (kc_env == 16 || (kc_env == 0 && K <= 16)) {
    dim3 gs((K + 15) / 16, batch);
    trsm_blocked_kernel<true, 16><<<gs, SolveCfg<16>::NT, SolveCfg<16>::kSmem, stream>>>(LU, ld, pencil_stride, n,
                                                                                        Y, ldy, ystride, K, pmap, klL, kuU);
    CIRR_CHECK_LAUNCH();
    trsm_blocked_kernel<false, 16><<<gs, SolveCfg<16>::NT, SolveCfg<16>::kSmem, stream>>>(LU, ld, pencil_stride, n,
                                                                                         Y, ldy, ystride, K, pmap, klL, kuU);
    CIRR_CHECK_LAUNCH();
  } else {
    dim3 gs((K + SKC - 1) / SKC, batch);
    trsm_blocked_kernel<true, 32><<<gs, SolveCfg<32>::NT, SolveCfg<32>::kSmem, stream>>>(LU, ld, pencil_stride, n,
                                                                                        Y, ldy, ystride, K, pmap, klL, kuU);
    CIRR_CHECK_LAUNCH();
    trsm_blocked_kernel<false, 32><<<gs, SolveCfg<32>::NT, SolveCfg<32>::kSmem, stream>>>(LU, ld, pencil_stride, n,
                                                                                         Y, ldy, ystride, K, pmap, klL, kuU);
    CIRR_CHECK_LAUNCH();
  }
  return moments_rows(ms, Y, ldy, ystride, n, K, 0, n, stream);
}

CIRR_API int cirr_zgetrs_batched(const cplx* LU, int n, long long ld, long long pencil_stride, int batch,
                                 const int* perm, const cplx* R, long long ldr, long long rstride,
                                 const int* rhs_of, int K, cplx* Y, long long ldy, long long ystride,
                                 const cplx* Dinv, cudaStream_t stream) {
  return getrs_impl(LU, n, ld, pencil_stride, batch, batch, nullptr, perm, R, ldr, rstride, rhs_of, K, Y, ldy,
                    ystride, Dinv, stream);
}

// The same solves for any subset of the factors: entry j uses factor
// pencil_of[j] (device int32, each < nfac), so contours that are not adjacent
// in the factor buffer still share one call (and one launch per GEMM step).
CIRR_API int cirr_zgetrs_gather(const cplx* LU, int n, long long ld, long long pencil_stride, int nfac,
                                const int* pencil_of, int batch, const int* perm, const cplx* R, long long ldr,
                                long long rstride, const int* rhs_of, int K, cplx* Y, long long ldy,
                                long long ystride, const cplx* Dinv, cudaStream_t stream) {
  if (pencil_of == nullptr) return CIRR_EINVAL;
  return getrs_impl(LU, n, ld, pencil_stride, batch, nfac, pencil_of, perm, R, ldr, rstride, rhs_of, K, Y, ldy,
                    ystride, Dinv, stream);
}

// Solves + moments: cirr_zgetrs_batched / cirr_zgetrs_gather whose moment
// accumulation St[c] = sum_j coef[j*M+m] Y_j (cirr_moments' layout, M <= 16)
// runs inside the solve: on the blocked TMA path each 128-row block of every
// entry's Y is accumulated right after the backward step that finishes it
// (L2-resident), so Y is not re-read from HBM by a separate moment pass.
CIRR_API int cirr_zgetrs_moments(const cplx* LU, int n, long long ld, long long pencil_stride, int nfac,
                                 const int* pencil_of, int batch, const int* perm, const cplx* R, long long ldr,
                                 long long rstride, const int* rhs_of, int K, cplx* Y, long long ldy,
                                 long long ystride, const cplx* Dinv, const cplx* coef, int M, const int* off,
                                 int n_sets, cplx* St, long long ld_st, long long sstride, cudaStream_t stream) {
  if (coef == nullptr || off == nullptr || St == nullptr) return CIRR_EINVAL;
  const MomentSpec ms{coef, M, off, n_sets, St, ld_st, sstride};
  return getrs_impl(LU, n, ld, pencil_stride, batch, pencil_of ? nfac : batch, pencil_of, perm, R, ldr, rstride,
                    rhs_of, K, Y, ldy, ystride, Dinv, stream, &ms);
}

// cirr_zgetrs_moments / cirr_zgetrs_gather / cirr_zgetrs_batched in one entry
// with the factors' bandwidths: klL (L below the diagonal: max(kl, the lbw of
// cirr_zgetrf_band)) and kuU (U above it: kl + ku); -1 = dense.  pencil_of
// NULL: entry j uses factor j; coef NULL: no moments.
CIRR_API int cirr_zgetrs_band(const cplx* LU, int n, long long ld, long long pencil_stride, int nfac,
                              const int* pencil_of, int batch, const int* perm, const cplx* R, long long ldr,
                              long long rstride, const int* rhs_of, int K, cplx* Y, long long ldy, long long ystride,
                              const cplx* Dinv, const cplx* coef, int M, const int* off, int n_sets, cplx* St,
                              long long ld_st, long long sstride, int klL, int kuU, cudaStream_t stream) {
  if (coef != nullptr && (off == nullptr || St == nullptr)) return CIRR_EINVAL;
  const MomentSpec ms{coef, M, off, n_sets, St, ld_st, sstride};
  return getrs_impl(LU, n, ld, pencil_stride, batch, pencil_of ? nfac : batch, pencil_of, perm, R, ldr, rstride,
                    rhs_of, K, Y, ldy, ystride, Dinv, stream, coef ? &ms : nullptr, klL, kuU);
}

// Moment rows [row_lo, row_hi) of n_sets contours (rows past n are skipped):
// pencils off[c] .. off[c+1]-1 belong to contour c; coef[j*M + m] = w_j zeta_j^m.
// Output St[c] is (M*K) x n row-major (row m*K+col = column col of S_m), ld
// ld_st, stride sstride.  Up to 16 moments per launch (MAXM).
static int launch_moments(const cplx* Y, long long ldy, long long ystride, int n, int K, const cplx* coef, int M,
                          const int* off, int n_sets, cplx* St, long long ld_st, long long sstride, int row_lo,
                          int row_hi, cudaStream_t stream) {
  if (row_hi > n) row_hi = n;
  if (row_hi <= row_lo) return 0;
  // windows of a solve (<= 128 rows) use 8-row tiles so the launch still has
  // enough CTAs; whole-matrix calls use 32-row tiles (same sums, same order)
  const bool win = row_hi - row_lo <= 128;
  const int TR = win ? 8 : MTR;
  dim3 g((K + MTC - 1) / MTC, (row_hi - row_lo + TR - 1) / TR, n_sets);
#define CIRR_MOM(MMv, RQv) \
  moments_kernel<MMv, RQv><<<g, 256, 0, stream>>>(Y, ldy, ystride, n, K, coef, M, off, St, ld_st, sstride, row_lo)
  if (win) {
    if (M <= 1) CIRR_MOM(1, 1);
    else if (M <= 2) CIRR_MOM(2, 1);
    else if (M <= 4) CIRR_MOM(4, 1);
    else if (M <= 8) CIRR_MOM(8, 1);
    else CIRR_MOM(16, 1);
  } else {
    if (M <= 1) CIRR_MOM(1, 4);
    else if (M <= 2) CIRR_MOM(2, 4);
    else if (M <= 4) CIRR_MOM(4, 4);
    else if (M <= 8) CIRR_MOM(8, 4);
    else CIRR_MOM(16, 4);
  }
#undef CIRR_MOM
  CIRR_CHECK_LAUNCH();
  return 0;
}

// Moment blocks of n_sets contours over all n rows (see launch_moments).
CIRR_API int cirr_moments(const cplx* Y, long long ldy, long long ystride, int n, int K, const cplx* coef,
                          int M, const int* off, int n_sets, cplx* St, long long ld_st, long long sstride,
                          cudaStream_t stream) {
  if (n <= 0 || K < 0 || M < 1 || M > MAXM || n_sets <= 0) return CIRR_EINVAL;
  if (K == 0) return 0;
  return launch_moments(Y, ldy, ystride, n, K, coef, M, off, n_sets, St, ld_st, sstride, 0, n, stream);
}
