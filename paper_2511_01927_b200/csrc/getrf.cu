// K2: batched blocked complex128 LU with partial pivoting (P M = L U).
//
// Replaces linalg.py:55-71 (`spla.splu` on z*B - A + the pivot test).  Per
// panel step k (width NB): panel2_kernel factors the m x NB panel in place
// (one CTA per pencil; IB-wide sub-panels with a block-argmax pivot search,
// then a TRSM+GEMM update of the rest of the panel), swap_kernel applies the
// panel's interchanges outside it, trsm_kernel forms U12 = L11^-1 A12, and the
// trailing update A22 -= L21 U12 runs on the FP64 tensor pipe (gemm.cuh,
// DMMA).  Pivoting follows LAPACK zgetrf (izamax on |re|+|im|, first index on
// ties).  The factorisation also reports per pencil min_i |U_ii| (the
// reference's singular-shift test, linalg.py:68-70) and LAPACK-style info.
#include "common.cuh"
#include <cstdlib>
#include "gemm.cuh"
#include "lu_gemm.cuh"
#include "ozaki.cuh"

namespace {

constexpr int NB = 64;      // panel width
constexpr int IB = 8;       // sub-panel width inside the panel kernel

// Panel factorisation (one CTA per pencil factors the m x 64 panel in 8-column
// sub-panels; LAPACK zgetf2 arithmetic and pivoting).  Every pass over the panel
// is coalesced along rows: the 8-column sub-panel update maps 8 lanes to one
// row (128 contiguous bytes), the update of the columns right of the
// sub-panel maps 16 lanes to one row, and the pivot search of column c+1 is
// fused into the pass that updates it (argmax of |re|+|im|, first index on
// ties, as LAPACK izamax).  Only the first column of a panel needs a strided
// search.  The first version issued one 16-byte load per thread per row, which
// made the L1 tag stage the limit (82 % L1/TEX throughput in ncu; the first
// version of this kernel, replaced in round 1).
constexpr int PT2 = 512;

__device__ __forceinline__ void arg_better(double& best, int& bi, double ov, int oi) {
  if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
}

// CTA-wide argmax of (best, bi); result valid in every thread.
template <int PW2>
__device__ __forceinline__ int block_argmax(double best, int bi, double* rv, int* ri) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    arg_better(best, bi, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, bi, o));
  if (lane == 0) { rv[wid] = best; ri[wid] = bi; }
  __syncthreads();
  best = lane < PW2 ? rv[lane] : -1.0;
  bi = lane < PW2 ? ri[lane] : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    arg_better(best, bi, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, bi, o));
  return bi;
}

template <int PTT>
__global__ void __launch_bounds__(PTT, PTT == 32 ? 16 : (PTT == 64 ? 8 : (PTT == 128 ? 4 : 1))) panel2_kernel(cplx* __restrict__ P, int n, long long ld, long long pstride,
                                                     int k, int jb, int* __restrict__ ipiv,
                                                     double* __restrict__ minpiv, int* __restrict__ info, int rend,
                                                     int* __restrict__ lbw) {
  // rows [k, rend) can be nonzero in the panel columns (rend = n for a dense
  // pencil, k + jb + kl for a banded one); the rows below are exact zeros there
  // and stay so, so they are skipped.  ipiv is indexed with the full order n.
  constexpr int PW2 = PTT / 32;
  __shared__ double rv[PW2];
  __shared__ int ri[PW2];
  __shared__ cplx prow[NB];       // pivot row over the panel columns (after the swap)
  __shared__ cplx ublk[IB][NB];   // U rows of the sub-panel, for the rest update
  cplx* A = P + (long long)blockIdx.x * pstride;
  int* piv = ipiv + (long long)blockIdx.x * n;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double mp = minpiv[blockIdx.x];
  int inf = info[blockIdx.x];
  // candidate for the next pivot column: strided search of column k once per panel
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int r = k + tid; r < rend; r += PTT) arg_better(best, bi, cabs1(A[(long long)r * ld + k]), r);

  for (int c0 = 0; c0 < jb; c0 += IB) {
    const int ib = min(IB, jb - c0);
    for (int c = c0; c < c0 + ib; ++c) {
      const int row0 = k + c;
      int p = block_argmax<PW2>(best, bi, rv, ri);
      if (p >= rend) p = row0;  // empty candidate set cannot happen for row0 < n; keep LAPACK-safe
      if (tid == 0) piv[row0] = p;
      // swap rows row0 <-> p over the panel width; prow = the new row0
      for (int cc = tid; cc < jb; cc += PTT) {
        cplx* x = A + (long long)row0 * ld + k + cc;
        const cplx xv = *x;
        if (p != row0) {
          cplx* y = A + (long long)p * ld + k + cc;
          const cplx yv = *y;
          *x = yv;
          *y = xv;
          prow[cc] = yv;
          // an L entry of an earlier column of this panel moving down
          if (lbw != nullptr && cc < c && (xv.x != 0.0 || xv.y != 0.0)) atomicMax(lbw + blockIdx.x, p - (k + cc));
        } else {
          prow[cc] = xv;
        }
      }
      __syncthreads();
      const cplx pv = prow[c];
      if (tid == 0) {
        const double a = cabs(pv);
        mp = fmin(mp, a);
        if (a == 0.0 && inf == 0) inf = row0 + 1;
      }
      const bool nz = (pv.x != 0.0 || pv.y != 0.0);
      const cplx rp = nz ? crecip(pv) : cmk(0.0, 0.0);
      // scale column c and rank-1 update of columns (c, c0+ib): 8 lanes per row
      const int g = lane & 7, cl = c - c0;
      const bool upd = g > cl && g < ib;
      const cplx u = upd ? prow[c0 + g] : cmk(0.0, 0.0);
      const bool track = (g == cl + 1) && (g < ib);
      best = -1.0;
      bi = 0x7fffffff;
      constexpr int RSTEP = 4 * PW2;  // rows per CTA pass of one row group
      constexpr int RU = 8;           // row groups in flight per thread
      for (int rb = row0 + 1 + wid * 4; rb < rend; rb += RU * RSTEP) {
        cplx v[RU];
        bool act[RU];
#pragma unroll
        for (int q = 0; q < RU; ++q) {
          const int r = rb + q * RSTEP + (lane >> 3);
          act[q] = r < rend;
          v[q] = (act[q] && g >= cl && g < ib) ? A[(long long)r * ld + k + c0 + g] : cmk(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < RU; ++q) {
          const int r = rb + q * RSTEP + (lane >> 3);
          const cplx lraw = cmk(__shfl_sync(0xffffffffu, v[q].x, (lane & ~7) + cl),
                                __shfl_sync(0xffffffffu, v[q].y, (lane & ~7) + cl));
          const cplx l = nz ? cmul(lraw, rp) : lraw;
          if (act[q]) {
            cplx* dst = A + (long long)r * ld + k + c0 + g;
            if (g == cl) {
              *dst = l;
            } else if (upd) {
              cplx w = v[q];
              cfms(w, l, u);
              *dst = w;
              if (track) arg_better(best, bi, cabs1(w), r);
            }
          }
        }
      }
      __syncthreads();
    }
    // columns right of the sub-panel: [k+c0+ib, k+jb)
    const int nr = jb - c0 - ib;
    if (nr > 0) {
      const int r0 = k + c0;
      // U rows r0..r0+ib-1: forward substitution with the unit-lower L block
      for (int cc = tid; cc < nr; cc += PTT) {
        const int colg = k + c0 + ib + cc;
        cplx uu[IB];
        for (int i = 0; i < ib; ++i) {
          cplx v = A[(long long)(r0 + i) * ld + colg];
          for (int l2 = 0; l2 < i; ++l2) cfms(v, A[(long long)(r0 + i) * ld + k + c0 + l2], uu[l2]);
          uu[i] = v;
          A[(long long)(r0 + i) * ld + colg] = v;
          ublk[i][cc] = v;
        }
      }
      __syncthreads();
      // rows below: A[r][rest] -= L[r][c0:c0+ib] U, 16 lanes per row; fused
      // argmax of the first rest column (the next sub-panel's pivot column)
      const int h = lane >> 4, q16 = lane & 15;
      best = -1.0;
      bi = 0x7fffffff;
      for (int rA = r0 + ib + wid * 2 + h; rA < rend; rA += 4 * PW2) {
        // two rows per thread (rA and rA + 2*PW2): all their loads in flight together
        const int rr2[2] = {rA, rA + 2 * PW2};
        cplx l[2][IB], v[2][4];
#pragma unroll
        for (int u2 = 0; u2 < 2; ++u2) {
          const bool ok = rr2[u2] < rend;
          const cplx* lr = A + (long long)rr2[u2] * ld + k + c0;
#pragma unroll
          for (int i = 0; i < IB; ++i) l[u2][i] = (ok && i < ib) ? lr[i] : cmk(0.0, 0.0);
          const cplx* src = lr + ib;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int cc = q16 + 16 * t;
            v[u2][t] = (ok && cc < nr) ? src[cc] : cmk(0.0, 0.0);
          }
        }
#pragma unroll
        for (int u2 = 0; u2 < 2; ++u2) {
          if (rr2[u2] >= rend) continue;
          cplx* dst = A + (long long)rr2[u2] * ld + k + c0 + ib;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int cc = q16 + 16 * t;
            if (cc < nr) {
#pragma unroll
              for (int i = 0; i < IB; ++i)
                if (i < ib) cfms(v[u2][t], l[u2][i], ublk[i][cc]);
              dst[cc] = v[u2][t];
              if (cc == 0) arg_better(best, bi, cabs1(v[u2][t]), rr2[u2]);
            }
          }
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    minpiv[blockIdx.x] = mp;
    info[blockIdx.x] = inf;
  }
}

// Apply interchanges ipiv[k .. k+jb) to the columns outside the panel: all of
// [0, k) (the L part, LAPACK convention) and [k + jb, cend) (cend = n dense,
// k + jb + kl + ku banded: U's fill-in bound).  lbw (per pencil, optional)
// records max (row - col) over the nonzero L entries the swaps move: with
// row interchanges an L entry can end up more than kl below the diagonal, and
// the band-limited solves need L's final lower bandwidth.
__global__ void swap_kernel(cplx* __restrict__ P, int n, long long ld, long long pstride, int k, int jb,
                            const int* __restrict__ ipiv, int cend, int* __restrict__ lbw, int kl) {
  const int other = k + (cend - k - jb);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  // banded: the rows swapped here (<= k + jb + kl) have their L entries in
  // columns >= k - max(kl, lbw) (lbw as of this launch: the earlier panels'
  // drift and this panel's own, recorded before); the columns left of that
  // are zeros in both rows
  const int lmin = (lbw != nullptr && kl < n - 1) ? max(0, k - max(kl, lbw[blockIdx.y])) : 0;
  int bw = 0;
  if (t < other && (t >= k || t >= lmin)) {
    const int col = t < k ? t : t + jb;
    cplx* A = P + (long long)blockIdx.y * pstride;
    const int* piv = ipiv + (long long)blockIdx.y * n;
    for (int i = 0; i < jb; ++i) {
      const int r1 = k + i, r2 = piv[k + i];
      if (r1 != r2) {
        cplx* x = A + (long long)r1 * ld + col;
        cplx* y = A + (long long)r2 * ld + col;
        const cplx tt = *x, yy = *y;
        *x = yy;
        *y = tt;
        if (col < k) {
          if (tt.x != 0.0 || tt.y != 0.0) bw = max(bw, r2 - col);
          if (yy.x != 0.0 || yy.y != 0.0) bw = max(bw, r1 - col);
        }
      }
    }
  }
  if (lbw != nullptr) {
    bw = __reduce_max_sync(0xffffffffu, bw);
    if ((threadIdx.x & 31) == 0 && bw > 0) atomicMax(lbw + blockIdx.y, bw);
  }
}

// U12 = L11^{-1} A12 for a 32-column chunk; L11 unit lower (jb x jb).
constexpr int TC = 32;
constexpr int kTrsmSmem = (NB * (NB + 1) + NB * (TC + 1)) * 16;
__global__ void __launch_bounds__(256) trsm_kernel(cplx* __restrict__ P, int n, long long ld,
                                                   long long pstride, int k, int jb) {
  extern __shared__ cplx tsm[];
  cplx(*L)[NB + 1] = reinterpret_cast<cplx(*)[NB + 1]>(tsm);
  cplx(*X)[TC + 1] = reinterpret_cast<cplx(*)[TC + 1]>(tsm + NB * (NB + 1));
  cplx* A = P + (long long)blockIdx.y * pstride;
  const int c0 = k + jb + blockIdx.x * TC;
  const int nc = min(TC, n - c0);
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    int r = e / jb, c = e % jb;
    L[r][c] = A[(long long)(k + r) * ld + k + c];
  }
  for (int e = threadIdx.x; e < jb * TC; e += blockDim.x) {
    int r = e / TC, c = e % TC;
    X[r][c] = c < nc ? A[(long long)(k + r) * ld + c0 + c] : cmk(0.0, 0.0);
  }
  __syncthreads();
  const int c = threadIdx.x % TC, g = threadIdx.x / TC, ng = blockDim.x / TC;
  for (int i = 0; i < jb - 1; ++i) {
    const cplx xi = X[i][c];
    for (int r = i + 1 + g; r < jb; r += ng) cfms(X[r][c], L[r][i], xi);
    __syncthreads();
  }
  for (int e = threadIdx.x; e < jb * TC; e += blockDim.x) {
    int r = e / TC, cc = e % TC;
    if (cc < nc) A[(long long)(k + r) * ld + c0 + cc] = X[r][cc];
  }
}

// Linv[b] = L11^{-1} for the unit-lower 64x64 diagonal block of panel step k
// (|l_ij| <= 1 under partial pivoting, so the explicit inverse is benign --
// the MAGMA trtri+gemm approach).  U12 = Linv A12 then runs on the TMA GEMM.
// Column j of X = L^-1 by forward substitution, x_i = -sum_{j<=k<i} L_ik x_k,
// four threads per column splitting the k sum (two shuffles combine it): no
// CTA barrier inside the substitution, and L, X packed lower-triangular in
// shared memory (66 KB, three CTAs per SM).  The first version ran one
// row-update sweep per i with a CTA barrier each (63 barriers, 133 KB, one
// CTA per SM): 2.1 ms per launch on config 2's 8192 pencils.
constexpr int kLinvSmem = NB * (NB + 1) * 16;   // two packed triangles
__device__ __forceinline__ int tri(int i) { return i * (i + 1) / 2; }
__global__ void __launch_bounds__(256) linv_kernel(const cplx* __restrict__ P, long long ld, long long pstride, int k,
                                                   cplx* __restrict__ Linv) {
  extern __shared__ cplx lsm[];
  cplx* Lp = lsm;                       // L[i][c], c <= i
  cplx* Xp = lsm + NB * (NB + 1) / 2;   // X[i][c], c <= i
  const cplx* A = P + (long long)blockIdx.x * pstride;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    if (c <= r) {
      Lp[tri(r) + c] = A[(long long)(k + r) * ld + k + c];
      Xp[tri(r) + c] = cmk(r == c ? 1.0 : 0.0, 0.0);
    }
  }
  __syncthreads();
  const int j = threadIdx.x >> 2, q = threadIdx.x & 3;
  for (int i = 1; i < NB; ++i) {
    double sr = 0.0, si = 0.0;
    const cplx* Li = Lp + tri(i);
    for (int kk = q; kk < i; kk += 4) {
      if (kk >= j) {
        const cplx a = Li[kk], x = Xp[tri(kk) + j];
        sr = fma(a.x, x.x, sr);
        sr = fma(-a.y, x.y, sr);
        si = fma(a.x, x.y, si);
        si = fma(a.y, x.x, si);
      }
    }
    sr += __shfl_xor_sync(0xffffffffu, sr, 1);
    si += __shfl_xor_sync(0xffffffffu, si, 1);
    sr += __shfl_xor_sync(0xffffffffu, sr, 2);
    si += __shfl_xor_sync(0xffffffffu, si, 2);
    if (q == 0 && i > j) Xp[tri(i) + j] = cmk(-sr, -si);
    __syncwarp();
  }
  __syncthreads();
  cplx* out = Linv + (long long)blockIdx.x * NB * NB;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    out[e] = c <= r ? Xp[tri(r) + c] : cmk(0.0, 0.0);
  }
}

// perm[i] = source row of row i of P*M (composition of the ipiv interchanges).
__global__ void perm_kernel(const int* __restrict__ ipiv, int* __restrict__ perm, int n) {
  extern __shared__ int sp[];
  const int* piv = ipiv + (long long)blockIdx.x * n;
  int* out = perm + (long long)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sp[i] = i;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      int p = piv[i];
      if (p != i) { int t = sp[i]; sp[i] = sp[p]; sp[p] = t; }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = sp[i];
}

__global__ void init_kernel(double* minpiv, int* info, int batch) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < batch) { minpiv[i] = INFINITY; info[i] = 0; }
}


}  // namespace

// In-place batched LU of `batch` complex n x n row-major matrices (stride
// pencil_stride elements, leading dimension ld).  Outputs ipiv (batch x n,
// 0-based LAPACK-style interchanges), perm (batch x n, row permutation),
// minpiv (min_i |U_ii|) and info (first exact zero pivot, 1-based, or 0).
// One CTA per pencil.  512 threads per CTA (measured best at n = 4096, and at
// n = 512 / 2304 with 32 / 96 pencils); for large batches of short panels
// (config 2: 8192 pencils, n = 256) the per-column latency chain dominates and
// 128-thread CTAs keep ~4x more pencils in flight per SM (4 CTAs per SM at 128 registers; LU 61.5 -> 38.1 ms).
// CIRR_PANEL_T overrides: 128 / 256 / 512.
static int launch_panel(cplx* pencils, int n, long long ld, long long pstride, int batch, int k, int jb, int* ipiv,
                        double* minpiv, int* info, int rend, int* lbw, cudaStream_t stream) {
  static const int env_t = getenv("CIRR_PANEL_T") ? atoi(getenv("CIRR_PANEL_T")) : 0;
  const int m = rend - k;   // rows the panel can have nonzero
  const int t = env_t > 0 ? env_t : (batch >= 1024 ? (m <= 128 ? 32 : (m <= 512 ? 128 : PT2)) : PT2);
  if (t == 32)
    panel2_kernel<32><<<batch, 32, 0, stream>>>(pencils, n, ld, pstride, k, jb, ipiv, minpiv, info, rend, lbw);
  else if (t == 64)
    panel2_kernel<64><<<batch, 64, 0, stream>>>(pencils, n, ld, pstride, k, jb, ipiv, minpiv, info, rend, lbw);
  else if (t == 128)
    panel2_kernel<128><<<batch, 128, 0, stream>>>(pencils, n, ld, pstride, k, jb, ipiv, minpiv, info, rend, lbw);
  else if (t == 256)
    panel2_kernel<256><<<batch, 256, 0, stream>>>(pencils, n, ld, pstride, k, jb, ipiv, minpiv, info, rend, lbw);
  else panel2_kernel<PT2><<<batch, PT2, 0, stream>>>(pencils, n, ld, pstride, k, jb, ipiv, minpiv, info, rend, lbw);
  CIRR_CHECK_LAUNCH();
  return 0;
}

// Workspace for cirr_zgetrf_batched (L11^{-1} blocks); 0 disables that path.
CIRR_API long long cirr_zgetrf_ws_bytes(int n, int batch) { return (long long)batch * NB * NB * 16 + 256; }

// Banded pencils (kl sub-, ku superdiagonals, the stencil configs 1/2/3/5)
// run the same kernels on the band only: the panel's rows stop at
// k + jb + kl, the interchanges and the U blocks at column k + jb + kl + ku
// (U's fill-in bound), the trailing updates cover the kl rows x (kl + ku)
// columns that can be nonzero.  Everything outside is an exact zero that the
// full LU would only add zeros to, so the factors are bitwise those of the
// dense LU.  kl = ku = n - 1 is the dense LU.  lbw (per pencil, zeroed by the
// caller, optional) receives L's final lower bandwidth beyond kl.
static int getrf_impl(cplx* pencils, int n, long long ld, long long pencil_stride, int batch, int kl, int ku,
                      int* ipiv, int* perm, double* minpiv, int* info, int* lbw, void* ws, cudaStream_t stream) {
  if (n <= 0 || batch <= 0 || ld < n || kl < 0 || ku < 0) return CIRR_EINVAL;
  kl = min(kl, n - 1);
  ku = min(ku, n - 1);
  // digit slices kept for earlier factors in this memory are stale now
  cirr::ozaki_invalidate(pencils, ((long long)(batch - 1) * pencil_stride + (long long)(n - 1) * ld + n) * 16);
  auto rend = [&](int k, int jb) { return (int)min((long long)n, (long long)k + jb + kl); };
  auto cend = [&](int k, int jb) { return (int)min((long long)n, (long long)k + jb + kl + ku); };
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmSmem);
    attr = true;
  }
  init_kernel<<<(batch + 255) / 256, 256, 0, stream>>>(minpiv, info, batch);
  CIRR_CHECK_LAUNCH();
  cirr::PencilMaps maps;
  const bool use_tma = cirr::encode_pencil_maps(maps, pencils, n, ld, pencil_stride, batch) == 0;
  cplx* linv = reinterpret_cast<cplx*>(ws);
  CUtensorMap mapL;
  const bool use_linv = use_tma && linv != nullptr &&
                        cirr::encode_a_map(&mapL, linv, NB, NB, batch, NB, (long long)NB * NB) == 0;
  if (use_linv) {
    static bool la = false;
    if (!la) {
      cudaFuncSetAttribute(linv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLinvSmem);
      la = true;
    }
  }
  int k0 = 0;
  if (use_linv && use_tma && n >= 256) {
    // Multi-level blocking: steps of W = PB x 64 columns made of PB 64-column
    // panels, so the big trailing update runs with k = W (fewer C-tile round
    // trips per flop: cuBLAS batched ZGEMM on these shapes goes 32.8 / 34.6 /
    // 35.7 TF/s at k = 64 / 128 / 256).  Inside a block the panels are
    // left-looking: just before panel i is factored, its columns receive the
    // updates of panels 0..i-1 of the block (one GEMM, k = 64 i); after it is
    // factored, its rows right of it receive the same deferred updates and
    // L_ii^-1 (U rows, in place).  Row interchanges of a panel go to every
    // column outside it and commute with the deferred row-wise updates.
    // CIRR_LU_PB overrides the panels per step (config 3, n = 2304: 119.0 /
    // 119.6 / 119.1 ms at 8 / 4 / 6 -- the 256-column tail costs nothing;
    // config 5: 5.44 s at 8 vs 5.50 s at 4)
    // Banded pencils (kl + ku below n / 2) take single 64-column steps: their
    // trailing windows are only kl x (kl + ku), so the k = W update saves
    // little, and the left-looking updates inside a step would sweep the full
    // kl + 64 panel rows once per panel (config 5: LU 215 -> 154 ms, config 3
    // 15.2 -> 11.2 ms, config 2 42 -> 39 ms at PB = 1).
    static const int pb_env = getenv("CIRR_LU_PB") ? atoi(getenv("CIRR_LU_PB")) : 0;
    const bool banded = (long long)kl + ku + 2 <= n / 2;
    const int PB = pb_env > 0 ? pb_env : (banded ? 1 : (n >= 2048 ? 8 : (n >= 1024 ? 4 : 2)));
    const int W = PB * NB;
    for (; k0 + W <= n; k0 += W) {
      const int k = k0, rest = n - k0 - W;
      for (int i = 0; i < PB; ++i) {
        const int ki = k + i * NB;
        const int re = rend(ki, NB), ce = cend(ki, NB);
        if (i > 0)  // this panel's columns: A[ki:re, ki:ki+64] -= L[ki:re, k:ki] U[k:ki, ki:ki+64]
          CIRR_TRY(cirr::zgemm_sub_maps(maps.a, maps.b, maps.c, re - ki, NB, i * NB, batch, ki, k, k, ki, ki, ki,
                                        pencils, ld, pencil_stride, stream));
        CIRR_TRY(launch_panel(pencils, n, ld, pencil_stride, batch, ki, NB, ipiv, minpiv, info, re, lbw, stream));
        {
          dim3 g((ki + ce - ki - NB + 255) / 256, batch);
          swap_kernel<<<g, 256, 0, stream>>>(pencils, n, ld, pencil_stride, ki, NB, ipiv, ce, lbw, kl);
          CIRR_CHECK_LAUNCH();
        }
        const int right = ce - ki - NB;  // columns right of this panel that can be nonzero
        if (right > 0) {
          linv_kernel<<<batch, 256, kLinvSmem, stream>>>(pencils, ld, pencil_stride, ki, linv);
          CIRR_CHECK_LAUNCH();
          if (i > 0)  // deferred updates of this panel's rows: A[ki:ki+64, ki+64:] -= L[ki:ki+64, k:ki] U[k:ki, ki+64:]
            CIRR_TRY(cirr::zgemm_sub_maps(maps.a, maps.b, maps.c, NB, right, i * NB, batch, ki, k, k, ki + NB, ki,
                                          ki + NB, pencils, ld, pencil_stride, stream));
          CIRR_TRY(cirr::zgemm_sub_maps(mapL, maps.b, maps.c, NB, right, NB, batch, 0, 0, ki, ki + NB, ki, ki + NB,
                                        pencils, ld, pencil_stride, stream, /*beta=*/0));
        }
      }
      if (rest > 0) {  // trailing update with k = W (rows/columns that can be nonzero)
        const int tm = rend(k, W) - k - W, tn = cend(k, W) - k - W;
        if (cirr::ozaki_enabled() && !banded && W >= 256 && cirr::ozaki_shape_ok(tm, tn, W)) {
          // int8 tensor cores (ozaki.cu): ~1.6x the DMMA kernel at this shape
          const cplx* a = pencils + (long long)(k + W) * ld + k;
          const cplx* b = pencils + (long long)k * ld + k + W;
          cplx* c = pencils + (long long)(k + W) * ld + k + W;
          CIRR_TRY(cirr::ozaki_zgemm_sub(a, ld, pencil_stride, b, ld, pencil_stride, c, ld, pencil_stride, tm, tn, W,
                                         batch, stream));
        } else {
          CIRR_TRY(cirr::zgemm_sub_maps(maps.a, maps.b, maps.c, tm, tn, W, batch, k + W, k, k, k + W, k + W, k + W,
                                        pencils, ld, pencil_stride, stream));
        }
      }
    }
  }
  for (int k = k0; k < n; k += NB) {
    const int jb = min(NB, n - k);
    const int re = rend(k, jb), ce = cend(k, jb);
    CIRR_TRY(launch_panel(pencils, n, ld, pencil_stride, batch, k, jb, ipiv, minpiv, info, re, lbw, stream));
    if (k + ce - k - jb > 0) {
      dim3 g((k + ce - k - jb + 255) / 256, batch);
      swap_kernel<<<g, 256, 0, stream>>>(pencils, n, ld, pencil_stride, k, jb, ipiv, ce, lbw, kl);
      CIRR_CHECK_LAUNCH();
    }
    const int rest = ce - k - jb;     // columns right of the panel that can be nonzero
    const int rrest = re - k - jb;    // rows below it that can be nonzero
    if (rest > 0) {
      if (use_linv && jb == NB) {
        // U12 = L11^{-1} A12 as a TMA/DMMA GEMM (each output tile reads exactly
        // the A12 tile it overwrites, so in place is safe)
        linv_kernel<<<batch, 256, kLinvSmem, stream>>>(pencils, ld, pencil_stride, k, linv);
        CIRR_CHECK_LAUNCH();
        CIRR_TRY(cirr::zgemm_sub_maps(mapL, maps.b, maps.c, NB, rest, NB, batch, 0, 0, k, k + jb, k, k + jb, pencils,
                                      ld, pencil_stride, stream, /*beta=*/0));
      } else {
        dim3 g2((rest + TC - 1) / TC, batch);
        trsm_kernel<<<g2, 256, kTrsmSmem, stream>>>(pencils, n, ld, pencil_stride, k, jb);
        CIRR_CHECK_LAUNCH();
      }
      if (jb % cirr::PBK == 0 && use_tma) {
        CIRR_TRY(cirr::zgemm_sub_maps(maps.a, maps.b, maps.c, rrest, rest, jb, batch, k + jb, k, k, k + jb, k + jb,
                                      k + jb, pencils, ld, pencil_stride, stream));
      } else if (rrest > 0) {
        cirr::GemmArgs ga{rrest, rest, jb, batch,
                          pencils + (long long)(k + jb) * ld + k, ld, pencil_stride,
                          pencils + (long long)k * ld + k + jb, ld, pencil_stride,
                          pencils + (long long)(k + jb) * ld + k + jb, ld, pencil_stride,
                          -1.0, 1};
        CIRR_TRY((cirr::gemm_launch<false, false>(ga, stream)));
      }
    }
  }
  if (perm) {
    size_t sm = sizeof(int) * (size_t)n;
    if (sm > 48 * 1024) cudaFuncSetAttribute(perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    perm_kernel<<<batch, 256, sm, stream>>>(ipiv, perm, n);
    CIRR_CHECK_LAUNCH();
  }
  return 0;
}

CIRR_API int cirr_zgetrf_batched(cplx* pencils, int n, long long ld, long long pencil_stride, int batch,
                                 int* ipiv, int* perm, double* minpiv, int* info, void* ws, cudaStream_t stream) {
  return getrf_impl(pencils, n, ld, pencil_stride, batch, n - 1, n - 1, ipiv, perm, minpiv, info, nullptr, ws,
                    stream);
}

// cirr_zgetrf_batched for pencils with kl sub- and ku superdiagonals (the
// union pattern of A and B, cirr_bandwidth); lbw: batch ints zeroed by the
// caller, each raised to the lower bandwidth the interchanges give L beyond kl
// (the solves take max(kl, lbw) and kl + ku).
CIRR_API int cirr_zgetrf_band(cplx* pencils, int n, long long ld, long long pencil_stride, int batch, int kl,
                              int ku, int* ipiv, int* perm, double* minpiv, int* info, int* lbw, void* ws,
                              cudaStream_t stream) {
  return getrf_impl(pencils, n, ld, pencil_stride, batch, kl, ku, ipiv, perm, minpiv, info, lbw, ws, stream);
}
