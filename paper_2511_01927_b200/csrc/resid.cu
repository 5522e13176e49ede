// K7 helpers: residual norms of Ritz pairs, column gathers and transposes.
//
// Replaces solvers.py:140-147 (_residuals: ||Ax - lam Bx|| / (||Ax|| +
// |lam| ||Bx||), zero denominator -> 1e-300) and the fancy indexing of
// solvers.py:196 (x = xs[:, keep]).  The GEMMs X = Q s, A X, B X run on the
// DMMA GEMM (gemm.cu).
#include "common.cuh"

namespace {

// res[b][i] for i < kdim[b]; AX, BX: n x kmax row-major per problem.
__global__ void __launch_bounds__(256) residual_kernel(const cplx* __restrict__ AX, const cplx* __restrict__ BX,
                                                       long long ld, long long stride, int n,
                                                       const cplx* __restrict__ lam, long long lstride,
                                                       const int* __restrict__ kdim, double* __restrict__ res,
                                                       long long rstride) {
  __shared__ double red[3][8];
  const int b = blockIdx.y, i = blockIdx.x;
  if (i >= kdim[b]) return;
  const cplx l = lam[(long long)b * lstride + i];
  const cplx* ax = AX + (long long)b * stride + i;
  const cplx* bx = BX + (long long)b * stride + i;
  double num = 0.0, na = 0.0, nb = 0.0;
  for (int r = threadIdx.x; r < n; r += 256) {
    const cplx a = ax[(long long)r * ld], bb = bx[(long long)r * ld];
    const cplx d = csub(a, cmul(l, bb));
    num += cabs2(d);
    na += cabs2(a);
    nb += cabs2(bb);
  }
  num = warp_sum(num); na = warp_sum(na); nb = warp_sum(nb);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { red[0][wid] = num; red[1][wid] = na; red[2][wid] = nb; }
  __syncthreads();
  if (threadIdx.x == 0) {
    num = na = nb = 0.0;
    for (int w = 0; w < 8; ++w) { num += red[0][w]; na += red[1][w]; nb += red[2][w]; }
    double den = sqrt(na) + cabs(l) * sqrt(nb);
    if (den == 0.0) den = 1e-300;
    res[(long long)b * rstride + i] = sqrt(num) / den;
  }
}

// out[b][r][c] = in[b][r][idx[b][c]]  for c < cnt[b] (r < n)
__global__ void gather_cols_kernel(const cplx* __restrict__ in, long long ldi, long long si,
                                   const int* __restrict__ idx, long long sidx, const int* __restrict__ cnt,
                                   int n, cplx* __restrict__ out, long long ldo, long long so) {
  const int b = blockIdx.z;
  const int r = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n || c >= cnt[b]) return;
  out[(long long)b * so + (long long)r * ldo + c] = in[(long long)b * si + (long long)r * ldi + idx[(long long)b * sidx + c]];
}

// out[b][j][i] = op(in[b][i][j]),  in: rows x cols
template <bool CONJ>
__global__ void transpose_kernel(const cplx* __restrict__ in, long long ldi, long long si, int rows, int cols,
                                 cplx* __restrict__ out, long long ldo, long long so) {
  __shared__ cplx tile[32][33];
  const int b = blockIdx.z;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const cplx* ip = in + (long long)b * si;
  cplx* op = out + (long long)b * so;
  for (int y = threadIdx.y; y < 32; y += 8) {
    int r = r0 + y, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[y][threadIdx.x] = ip[(long long)r * ldi + c];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    int c = c0 + y, r = r0 + threadIdx.x;
    if (r < rows && c < cols) {
      cplx v = tile[threadIdx.x][y];
      if (CONJ) v.y = -v.y;
      op[(long long)c * ldo + r] = v;
    }
  }
}

}  // namespace

CIRR_API int cirr_residuals(const cplx* AX, const cplx* BX, long long ld, long long stride, int n,
                            const cplx* lam, long long lstride, const int* kdim, int kmax, int nprob,
                            double* res, long long rstride, cudaStream_t stream) {
  if (n <= 0 || kmax <= 0 || nprob <= 0) return CIRR_EINVAL;
  dim3 g(kmax, nprob);
  residual_kernel<<<g, 256, 0, stream>>>(AX, BX, ld, stride, n, lam, lstride, kdim, res, rstride);
  CIRR_CHECK_LAUNCH();
  return 0;
}

CIRR_API int cirr_gather_cols(const cplx* in, long long ldi, long long si, const int* idx, long long sidx,
                              const int* cnt, int cmax, int n, int nprob, cplx* out, long long ldo, long long so,
                              cudaStream_t stream) {
  if (n <= 0 || nprob <= 0 || cmax < 0) return CIRR_EINVAL;
  if (cmax == 0) return 0;
  dim3 g((cmax + 127) / 128, n, nprob);
  gather_cols_kernel<<<g, 128, 0, stream>>>(in, ldi, si, idx, sidx, cnt, n, out, ldo, so);
  CIRR_CHECK_LAUNCH();
  return 0;
}

CIRR_API int cirr_transpose(int conj, const cplx* in, long long ldi, long long si, int rows, int cols, int batch,
                            cplx* out, long long ldo, long long so, cudaStream_t stream) {
  if (rows < 0 || cols < 0 || batch < 0) return CIRR_EINVAL;
  if (rows == 0 || cols == 0 || batch == 0) return 0;
  dim3 g((cols + 31) / 32, (rows + 31) / 32, batch);
  dim3 t(32, 8);
  if (conj) transpose_kernel<true><<<g, t, 0, stream>>>(in, ldi, si, rows, cols, out, ldo, so);
  else transpose_kernel<false><<<g, t, 0, stream>>>(in, ldi, si, rows, cols, out, ldo, so);
  CIRR_CHECK_LAUNCH();
  return 0;
}

namespace {
// out[b][r][c] = op_b(in[src[b]][r][col0[b] + c]),  op = conj when cj[b]
__global__ void copy_cols_kernel(const cplx* __restrict__ in, long long ldi, long long si, const int* __restrict__ src,
                                 const int* __restrict__ col0, const int* __restrict__ cj, int n, int K,
                                 cplx* __restrict__ out, long long ldo, long long so) {
  const int b = blockIdx.y;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * K) return;
  const int r = (int)(e / K), c = (int)(e % K);
  cplx v = in[(long long)src[b] * si + (long long)r * ldi + col0[b] + c];
  if (cj[b]) v.y = -v.y;
  out[(long long)b * so + (long long)r * ldo + c] = v;
}
}  // namespace

// Batched column-block copy with optional conjugation (builds the mirrored
// solutions Y_{N-1-j} = conj(M_j^-1 conj(R)) of the conjugate-pair variant).
CIRR_API int cirr_copy_cols(const cplx* in, long long ldi, long long si, const int* src, const int* col0,
                            const int* cj, int n, int K, int count, cplx* out, long long ldo, long long so,
                            cudaStream_t stream) {
  if (n <= 0 || K < 0 || count < 0) return CIRR_EINVAL;
  if (K == 0 || count == 0) return 0;
  dim3 g((unsigned)(((long long)n * K + 255) / 256), count);
  copy_cols_kernel<<<g, 256, 0, stream>>>(in, ldi, si, src, col0, cj, n, K, out, ldo, so);
  CIRR_CHECK_LAUNCH();
  return 0;
}

// --------------------------------------------------------------------------
// KDE sparsity for the contour construction upstream of the solve
// (kernels.py:38-67, contours.py:175-192):
// out[i] = sum_j exp(-coef * (ts[i] - eigs[j])^2), summed in j order.
namespace {
constexpr int KT = 256;
__global__ void __launch_bounds__(KT) kde_kernel(const double* __restrict__ ts, int nt,
                                                 const double* __restrict__ eigs, int ne, double coef,
                                                 double* __restrict__ out) {
  __shared__ double se[KT * 4];
  const int i = blockIdx.x * KT + threadIdx.x;
  const double t = i < nt ? ts[i] : 0.0;
  double acc = 0.0;
  for (int j0 = 0; j0 < ne; j0 += KT * 4) {
    const int cnt = min(KT * 4, ne - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += KT) se[e] = eigs[j0 + e];
    __syncthreads();
    for (int e = 0; e < cnt; ++e) {
      const double d = t - se[e];
      acc += exp(-coef * d * d);
    }
  }
  if (i < nt) out[i] = acc;
}
}  // namespace

CIRR_API int cirr_kde_eval(const double* ts, int nt, const double* eigs, int ne, double coef, double* out,
                           cudaStream_t stream) {
  if (nt < 0 || ne < 0) return CIRR_EINVAL;
  if (nt == 0) return 0;
  kde_kernel<<<(nt + KT - 1) / KT, KT, 0, stream>>>(ts, nt, eigs, ne, coef, out);
  CIRR_CHECK_LAUNCH();
  return 0;
}
