// K1: shifted-pencil assembly M_j = z_j B - A for every quadrature node.
//
// Replaces linalg.py:62 (`z * B - A`) and the scale of linalg.py:63
// (max |M_ij|, used by the singular-pivot test).  A and B are real float64,
// row-major; the pencils are complex128 row-major.  Each CTA reads one
// contiguous chunk of A and B once from HBM and writes it for a group of
// pencils (coalesced 16-byte stores), so the read traffic is ~1/group of the
// write traffic.  The arithmetic is written with __dmul_rn/__dsub_rn so the
// result is bitwise identical to numpy's (z*B - A): two roundings, no FMA.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 8;          // elements per thread per chunk
constexpr int kChunk = kThreads * kPerThread;
constexpr int kGroup = 8;              // pencils written per CTA

__global__ void __launch_bounds__(kThreads) assemble_kernel(
    const double* __restrict__ A, const double* __restrict__ B, int n, long long lda,
    const cplx* __restrict__ z, int nz, cplx* __restrict__ P, long long ldp, long long pstride,
    unsigned long long* __restrict__ maxabs_bits) {
  __shared__ double wmax[kThreads / 32][kGroup];
  const long long total = (long long)n * n;
  const long long base = (long long)blockIdx.x * kChunk;
  const int j0 = blockIdx.y * kGroup;
  double a[kPerThread], b[kPerThread];
  long long src[kPerThread], dst[kPerThread];
  bool ok[kPerThread];
#pragma unroll
  for (int e = 0; e < kPerThread; ++e) {
    long long idx = base + (long long)e * kThreads + threadIdx.x;
    ok[e] = idx < total;
    long long r = ok[e] ? idx / n : 0, c = ok[e] ? idx - r * n : 0;
    src[e] = r * lda + c;
    dst[e] = r * ldp + c;
    a[e] = ok[e] ? A[src[e]] : 0.0;
    b[e] = ok[e] ? B[src[e]] : 0.0;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int g = 0; g < kGroup; ++g) {
    const int j = j0 + g;
    if (j >= nz) break;
    const cplx zj = z[j];
    cplx* Pj = P + (long long)j * pstride;
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < kPerThread; ++e) {
      if (ok[e]) {
        cplx v = cmk(__dsub_rn(__dmul_rn(zj.x, b[e]), a[e]), __dmul_rn(zj.y, b[e]));
        Pj[dst[e]] = v;
        m = fmax(m, hypot(v.x, v.y));
      }
    }
    m = warp_max(m);
    if (lane == 0) wmax[wid][g] = m;
  }
  __syncthreads();
  if (threadIdx.x < kGroup && j0 + threadIdx.x < nz) {
    double m = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) m = fmax(m, wmax[w][threadIdx.x]);
    // non-negative doubles order like their bit patterns
    atomicMax(maxabs_bits + j0 + threadIdx.x, (unsigned long long)__double_as_longlong(m));
  }
}

// As assemble_kernel with the matrices of pencil j at a_ptrs[j], b_ptrs[j]
// (many GEPs in one launch, solve_multi_batch).  A CTA's group of pencils
// reloads its chunk of A and B only where the matrix changes from the
// previous pencil of the group.
__global__ void __launch_bounds__(kThreads) assemble_ptrs_kernel(
    const long long* __restrict__ a_ptrs, const long long* __restrict__ b_ptrs, int n, long long lda,
    const cplx* __restrict__ z, int nz, cplx* __restrict__ P, long long ldp, long long pstride,
    unsigned long long* __restrict__ maxabs_bits) {
  __shared__ double wmax[kThreads / 32][kGroup];
  const long long total = (long long)n * n;
  const long long base = (long long)blockIdx.x * kChunk;
  const int j0 = blockIdx.y * kGroup;
  double a[kPerThread], b[kPerThread];
  long long dst[kPerThread];
  const double* Acur = nullptr;
  const double* Bcur = nullptr;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int g = 0; g < kGroup; ++g) {
    const int j = j0 + g;
    if (j >= nz) break;
    const double* Aj = reinterpret_cast<const double*>(a_ptrs[j]);
    const double* Bj = reinterpret_cast<const double*>(b_ptrs[j]);
    if (Aj != Acur || Bj != Bcur) {
      Acur = Aj;
      Bcur = Bj;
#pragma unroll
      for (int e = 0; e < kPerThread; ++e) {
        const long long idx = base + (long long)e * kThreads + threadIdx.x;
        const bool ok = idx < total;
        const long long r = ok ? idx / n : 0, c = ok ? idx - r * n : 0;
        dst[e] = ok ? r * ldp + c : -1;
        a[e] = ok ? Aj[r * lda + c] : 0.0;
        b[e] = ok ? Bj[r * lda + c] : 0.0;
      }
    }
    const cplx zj = z[j];
    cplx* Pj = P + (long long)j * pstride;
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < kPerThread; ++e) {
      if (dst[e] >= 0) {
        cplx v = cmk(__dsub_rn(__dmul_rn(zj.x, b[e]), a[e]), __dmul_rn(zj.y, b[e]));
        Pj[dst[e]] = v;
        m = fmax(m, hypot(v.x, v.y));
      }
    }
    m = warp_max(m);
    if (lane == 0) wmax[wid][g] = m;
  }
  __syncthreads();
  if (threadIdx.x < kGroup && j0 + threadIdx.x < nz) {
    double m = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) m = fmax(m, wmax[w][threadIdx.x]);
    atomicMax(maxabs_bits + j0 + threadIdx.x, (unsigned long long)__double_as_longlong(m));
  }
}

// out[0] = max_ij |A_ij - A_ji|, out[1] = max_ij |A_ij| (as ordered bit patterns)
__global__ void symmetry_kernel(const double* __restrict__ A, int n, long long lda,
                                unsigned long long* __restrict__ out) {
  __shared__ double red[2][8];
  double d = 0.0, m = 0.0;
  const long long total = (long long)n * n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / n, c = e - r * n;
    const double a = A[r * lda + c];
    m = fmax(m, fabs(a));
    if (c > r) d = fmax(d, fabs(a - A[c * lda + r]));
  }
  d = warp_max(d);
  m = warp_max(m);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { red[0][wid] = d; red[1][wid] = m; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) { d = fmax(d, red[0][w]); m = fmax(m, red[1][w]); }
    d = fmax(d, red[0][0]);
    m = fmax(m, red[1][0]);
    atomicMax(out, (unsigned long long)__double_as_longlong(d));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(m));
  }
}

}  // namespace

// out[0] = max |A - A^T|, out[1] = max |A| for a real row-major matrix
// (the Hermitian test of sparse.py:83-87 on device).
CIRR_API int cirr_symmetry(const double* A, int n, long long lda, double* out, cudaStream_t stream) {
  if (n <= 0 || lda < n) return CIRR_EINVAL;
  cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(double), stream);
  if (e != cudaSuccess) return (int)e;
  long long total = (long long)n * n;
  int blocks = (int)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  symmetry_kernel<<<blocks, 256, 0, stream>>>(A, n, lda, reinterpret_cast<unsigned long long*>(out));
  CIRR_CHECK_LAUNCH();
  return 0;
}

// pencils[j] = z[j]*B - A (j < nz); maxabs[j] = max_ij |pencils[j]_ij|.
CIRR_API int cirr_assemble(const double* A, const double* B, int n, long long lda,
                           const cplx* z, int nz, cplx* pencils, long long ldp,
                           long long pencil_stride, double* maxabs, cudaStream_t stream) {
  if (n <= 0 || nz <= 0 || lda < n || ldp < n) return CIRR_EINVAL;
  cudaError_t e = cudaMemsetAsync(maxabs, 0, sizeof(double) * nz, stream);
  if (e != cudaSuccess) return (int)e;
  const long long total = (long long)n * n;
  dim3 grid((unsigned)((total + kChunk - 1) / kChunk), (unsigned)((nz + kGroup - 1) / kGroup));
  assemble_kernel<<<grid, kThreads, 0, stream>>>(A, B, n, lda, z, nz, pencils, ldp, pencil_stride,
                                                  reinterpret_cast<unsigned long long*>(maxabs));
  CIRR_CHECK_LAUNCH();
  return 0;
}

// cirr_assemble for nz pencils whose real A, B (n x n, ld lda) are at the
// device addresses a_ptrs[j], b_ptrs[j] (device int64[nz]): one launch for the
// pencils of many GEPs (solve_multi_batch), bitwise equal to cirr_assemble.
CIRR_API int cirr_assemble_ptrs(const long long* a_ptrs, const long long* b_ptrs, int n, long long lda,
                                const cplx* z, int nz, cplx* pencils, long long ldp, long long pencil_stride,
                                double* maxabs, cudaStream_t stream) {
  if (n <= 0 || nz <= 0 || lda < n || ldp < n || a_ptrs == nullptr || b_ptrs == nullptr) return CIRR_EINVAL;
  cudaError_t e = cudaMemsetAsync(maxabs, 0, sizeof(double) * nz, stream);
  if (e != cudaSuccess) return (int)e;
  const long long total = (long long)n * n;
  const long long gy = (nz + kGroup - 1) / kGroup;
  if (gy > 65535) return CIRR_EINVAL;
  dim3 grid((unsigned)((total + kChunk - 1) / kChunk), (unsigned)gy);
  assemble_ptrs_kernel<<<grid, kThreads, 0, stream>>>(a_ptrs, b_ptrs, n, lda, z, nz, pencils, ldp, pencil_stride,
                                                       reinterpret_cast<unsigned long long*>(maxabs));
  CIRR_CHECK_LAUNCH();
  return 0;
}

// --------------------------------------------------------------------------
// Complex-valued A and B (the reference's MatrixPencil holds complex128 CSR
// values, sparse.py:14-43; complex Hermitian pencils are valid input).
namespace {
__global__ void __launch_bounds__(kThreads) assemble_c_kernel(
    const cplx* __restrict__ A, const cplx* __restrict__ B, int n, long long lda,
    const cplx* __restrict__ z, int nz, cplx* __restrict__ P, long long ldp, long long pstride,
    unsigned long long* __restrict__ maxabs_bits) {
  __shared__ double wmax[kThreads / 32][kGroup];
  const long long total = (long long)n * n;
  const long long base = (long long)blockIdx.x * kChunk;
  const int j0 = blockIdx.y * kGroup;
  cplx a[kPerThread], b[kPerThread];
  long long dst[kPerThread];
  bool ok[kPerThread];
#pragma unroll
  for (int e = 0; e < kPerThread; ++e) {
    long long idx = base + (long long)e * kThreads + threadIdx.x;
    ok[e] = idx < total;
    long long r = ok[e] ? idx / n : 0, c = ok[e] ? idx - r * n : 0;
    dst[e] = r * ldp + c;
    a[e] = ok[e] ? A[r * lda + c] : cmk(0.0, 0.0);
    b[e] = ok[e] ? B[r * lda + c] : cmk(0.0, 0.0);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int g = 0; g < kGroup; ++g) {
    const int j = j0 + g;
    if (j >= nz) break;
    const cplx zj = z[j];
    cplx* Pj = P + (long long)j * pstride;
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < kPerThread; ++e) {
      if (ok[e]) {
        // numpy's complex product (rounded products, rounded sums, no FMA), then - A
        const double pr = __dsub_rn(__dmul_rn(zj.x, b[e].x), __dmul_rn(zj.y, b[e].y));
        const double pi = __dadd_rn(__dmul_rn(zj.x, b[e].y), __dmul_rn(zj.y, b[e].x));
        const cplx v = cmk(__dsub_rn(pr, a[e].x), __dsub_rn(pi, a[e].y));
        Pj[dst[e]] = v;
        m = fmax(m, hypot(v.x, v.y));
      }
    }
    m = warp_max(m);
    if (lane == 0) wmax[wid][g] = m;
  }
  __syncthreads();
  if (threadIdx.x < kGroup && j0 + threadIdx.x < nz) {
    double m = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) m = fmax(m, wmax[w][threadIdx.x]);
    atomicMax(maxabs_bits + j0 + threadIdx.x, (unsigned long long)__double_as_longlong(m));
  }
}

// out[0] = max_ij |A_ij - conj(A_ji)| (diagonal included), out[1] = max_ij |A_ij|
__global__ void hermitian_c_kernel(const cplx* __restrict__ A, int n, long long lda,
                                   unsigned long long* __restrict__ out) {
  __shared__ double red[2][8];
  double d = 0.0, m = 0.0;
  const long long total = (long long)n * n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / n, c = e - r * n;
    const cplx a = A[r * lda + c];
    m = fmax(m, cabs(a));
    if (c >= r) d = fmax(d, cabs(csub(a, cconj(A[c * lda + r]))));
  }
  d = warp_max(d);
  m = warp_max(m);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { red[0][wid] = d; red[1][wid] = m; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) { d = fmax(d, red[0][w]); m = fmax(m, red[1][w]); }
    d = fmax(d, red[0][0]);
    m = fmax(m, red[1][0]);
    atomicMax(out, (unsigned long long)__double_as_longlong(d));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(m));
  }
}
}  // namespace

// pencils[j] = z[j]*B - A for complex128 A, B (row-major, ld lda); maxabs as cirr_assemble.
CIRR_API int cirr_assemble_c(const cplx* A, const cplx* B, int n, long long lda, const cplx* z, int nz,
                             cplx* pencils, long long ldp, long long pencil_stride, double* maxabs,
                             cudaStream_t stream) {
  if (n <= 0 || nz <= 0 || lda < n || ldp < n) return CIRR_EINVAL;
  cudaError_t e = cudaMemsetAsync(maxabs, 0, sizeof(double) * nz, stream);
  if (e != cudaSuccess) return (int)e;
  const long long total = (long long)n * n;
  dim3 grid((unsigned)((total + kChunk - 1) / kChunk), (unsigned)((nz + kGroup - 1) / kGroup));
  assemble_c_kernel<<<grid, kThreads, 0, stream>>>(A, B, n, lda, z, nz, pencils, ldp, pencil_stride,
                                                    reinterpret_cast<unsigned long long*>(maxabs));
  CIRR_CHECK_LAUNCH();
  return 0;
}

// out[0] = max |A - A^H|, out[1] = max |A| for a complex128 row-major matrix
// (the Hermitian test of sparse.py:83-87 on device).
CIRR_API int cirr_hermitian_c(const cplx* A, int n, long long lda, double* out, cudaStream_t stream) {
  if (n <= 0 || lda < n) return CIRR_EINVAL;
  cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(double), stream);
  if (e != cudaSuccess) return (int)e;
  long long total = (long long)n * n;
  int blocks = (int)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  hermitian_c_kernel<<<blocks, 256, 0, stream>>>(A, n, lda, reinterpret_cast<unsigned long long*>(out));
  CIRR_CHECK_LAUNCH();
  return 0;
}

// --------------------------------------------------------------------------
// Band structure of the pencils (configs 1/2/3/5 are stencils stored dense):
// out[0] = max(i - j), out[1] = max(j - i) over the nonzero entries of the
// n x n matrix M (real f64 or complex128, row-major, ld), each raised with
// atomicMax (zero them first to start; call once per matrix for a union).
namespace {
__global__ void bandwidth_kernel(const double* __restrict__ M0, const long long* __restrict__ ptrs, int cw, int n,
                                 long long ld, int* __restrict__ out0) {
  // matrix blockIdx.y: M0 itself, or the one at ptrs[blockIdx.y]
  const double* M = ptrs ? reinterpret_cast<const double*>(ptrs[blockIdx.y]) : M0;
  int* out = out0 + 2 * blockIdx.y;
  int kl = 0, ku = 0;
  const long long total = (long long)n * n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), c = (int)(e - (long long)r * n);
    const double* x = M + ((long long)r * ld + c) * cw;
    const bool nz = x[0] != 0.0 || (cw == 2 && x[1] != 0.0);
    if (nz) {
      kl = max(kl, r - c);
      ku = max(ku, c - r);
    }
  }
  kl = __reduce_max_sync(0xffffffffu, kl);
  ku = __reduce_max_sync(0xffffffffu, ku);
  if ((threadIdx.x & 31) == 0) {
    if (kl > 0) atomicMax(out, kl);
    if (ku > 0) atomicMax(out + 1, ku);
  }
}
}  // namespace

CIRR_API int cirr_bandwidth(const void* M, int is_complex, int n, long long ld, int* out, cudaStream_t stream) {
  if (n <= 0 || ld < n || M == nullptr || out == nullptr) return CIRR_EINVAL;
  const long long total = (long long)n * n;
  const int blocks = (int)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  bandwidth_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const double*>(M), nullptr, is_complex ? 2 : 1, n, ld,
                                               out);
  CIRR_CHECK_LAUNCH();
  return 0;
}

// cirr_bandwidth for count matrices at the device addresses ptrs[i]
// (device int64[count]) in one launch: out[2 i], out[2 i + 1] (zeroed first).
CIRR_API int cirr_bandwidth_ptrs(const long long* ptrs, int count, int is_complex, int n, long long ld, int* out,
                                 cudaStream_t stream) {
  if (n <= 0 || ld < n || ptrs == nullptr || out == nullptr || count < 0 || count > 65535) return CIRR_EINVAL;
  if (count == 0) return 0;
  const long long total = (long long)n * n;
  long long bx = (total + 255) / 256;
  const long long cap = (148LL * 8 + count - 1) / count;
  if (bx > cap) bx = cap < 1 ? 1 : cap;
  bandwidth_kernel<<<dim3((unsigned)bx, count), 256, 0, stream>>>(nullptr, ptrs, is_complex ? 2 : 1, n, ld, out);
  CIRR_CHECK_LAUNCH();
  return 0;
}
