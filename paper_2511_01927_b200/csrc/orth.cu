// K4: rank-revealing orthonormalisation of the stacked moment block.
//
// Replaces linalg.py:107-119 (thin SVD of S, keep left singular vectors with
// sigma_i >= rel_tol * sigma_max).  One-sided (Hestenes) Jacobi is applied
// directly to the columns of S, stored as contiguous rows of St (c x n):
// pairs of columns are rotated until every normalised inner product is below
// 16 sqrt(n) eps.  On convergence the columns are U*Sigma with U orthonormal to
// working precision, so sigma_i = ||col_i|| resolves ratios down to ~1e-15 --
// needed because config 4's block has sigma_min/sigma_max ~ 2e-12 and a 1e-8
// cut loses most pairs (finding 7).  Gram-based
// CholeskyQR cannot resolve that.
//
// Rounds use the circle-method tournament (c/2 disjoint pairs per round) and
// run as ONE cooperative kernel with a software grid barrier between rounds;
// every reduction is a fixed-order block reduction, so results are
// bit-reproducible.
#include "common.cuh"

namespace {

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    unsigned gen = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) { __nanosleep(32); }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void rr_pair(int round, int k, int cp, int& p, int& q) {
  // circle method over cp (even) players; player cp-1 is fixed
  if (k == 0) {
    p = cp - 1;
    q = round;
  } else {
    p = (round + k) % (cp - 1);
    q = (round - k + (cp - 1)) % (cp - 1);
  }
}

constexpr int HT = 256;

__global__ void __launch_bounds__(HT) hestenes_kernel(cplx* __restrict__ W, long long ldw, long long wstride,
                                                       int n, int c, int nprob, unsigned* bar, int* counters,
                                                       int max_sweeps, double tol, int* sweeps_out) {
  __shared__ double red[4][HT / 32];
  const int cp = c + (c & 1);
  const int npairs = cp / 2;
  const long long items = (long long)nprob * npairs;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (blockIdx.x == 0 && threadIdx.x == 0) counters[(sweep + 1) & 1] = 0;
    for (int round = 0; round < cp - 1; ++round) {
      for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        const int prob = (int)(it / npairs), k = (int)(it % npairs);
        int p, q;
        rr_pair(round, k, cp, p, q);
        if (p >= c || q >= c) continue;
        if (p > q) { int t = p; p = q; q = t; }
        cplx* wp = W + (long long)prob * wstride + (long long)p * ldw;
        cplx* wq = W + (long long)prob * wstride + (long long)q * ldw;
        double a = 0.0, bb = 0.0, gr = 0.0, gi = 0.0;
        for (int i = threadIdx.x; i < n; i += HT) {
          cplx x = wp[i], y = wq[i];
          a += cabs2(x);
          bb += cabs2(y);
          cplx g = cconjmul(x, y);
          gr += g.x;
          gi += g.y;
        }
        a = warp_sum(a); bb = warp_sum(bb); gr = warp_sum(gr); gi = warp_sum(gi);
        __syncthreads();
        if (lane == 0) { red[0][wid] = a; red[1][wid] = bb; red[2][wid] = gr; red[3][wid] = gi; }
        __syncthreads();
        a = 0.0; bb = 0.0; gr = 0.0; gi = 0.0;
        for (int w = 0; w < HT / 32; ++w) { a += red[0][w]; bb += red[1][w]; gr += red[2][w]; gi += red[3][w]; }
        const double ag = hypot(gr, gi);
        if (a > 0.0 && bb > 0.0 && ag > tol * sqrt(a) * sqrt(bb)) {
          // [wp', wq'] = [wp, wq] [[c, s e^{i phi}], [-s e^{-i phi}, c]],  gamma = |gamma| e^{i phi}
          const double zeta = (bb - a) / (2.0 * ag);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = t * cs;
          const cplx e = cmk(gr / ag, gi / ag);
          const cplx se = cscale(e, sn);          // s e^{i phi}
          const cplx sec = cconj(se);             // s e^{-i phi}
          for (int i = threadIdx.x; i < n; i += HT) {
            cplx x = wp[i], y = wq[i];
            cplx nx = csub(cscale(x, cs), cmul(sec, y));
            cplx ny = cadd(cmul(se, x), cscale(y, cs));
            wp[i] = nx;
            wq[i] = ny;
          }
          if (threadIdx.x == 0) atomicAdd(counters + (sweep & 1), 1);
        }
      }
      grid_barrier(bar, gridDim.x);
    }
    const int rots = *((volatile int*)(counters + (sweep & 1)));
    grid_barrier(bar, gridDim.x);
    if (rots == 0) { ++sweep; break; }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

// sigma, descending order, kept count per problem (one CTA per problem).
__global__ void __launch_bounds__(1024) svd_finalize_kernel(const cplx* __restrict__ W, long long ldw,
                                                             long long wstride, int n, int c, double rel_tol,
                                                             double* __restrict__ sigma, int* __restrict__ order,
                                                             int* __restrict__ kept) {
  extern __shared__ double sg[];
  const int prob = blockIdx.x;
  const cplx* Wp = W + (long long)prob * wstride;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int row = wid; row < c; row += nw) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += cabs2(Wp[(long long)row * ldw + i]);
    s = warp_sum(s);
    if (lane == 0) sg[row] = sqrt(s);
  }
  __syncthreads();
  double smax = 0.0;
  for (int i = 0; i < c; ++i) smax = fmax(smax, sg[i]);
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    const double si = sg[i];
    int rank = 0;
    for (int j = 0; j < c; ++j) {
      const double sj = sg[j];
      rank += (sj > si) || (sj == si && j < i);
    }
    order[(long long)prob * c + rank] = i;
    sigma[(long long)prob * c + rank] = si;
  }
  if (threadIdx.x == 0) {
    int k = 0;
    if (smax > 0.0)
      for (int i = 0; i < c; ++i) k += sg[i] >= rel_tol * smax;
    kept[prob] = k;
  }
}

// Qt[prob][r][:] = W[prob][order[r]][:] / sigma[r]   for r < kept[prob]
__global__ void build_q_kernel(const cplx* __restrict__ W, long long ldw, long long wstride, int n, int c,
                               const double* __restrict__ sigma, const int* __restrict__ order,
                               const int* __restrict__ kept, cplx* __restrict__ Qt, long long ldq,
                               long long qstride) {
  const int prob = blockIdx.z, r = blockIdx.y;
  if (r >= kept[prob]) return;
  const int src = order[(long long)prob * c + r];
  const double inv = 1.0 / sigma[(long long)prob * c + r];
  const cplx* w = W + (long long)prob * wstride + (long long)src * ldw;
  cplx* q = Qt + (long long)prob * qstride + (long long)r * ldq;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    q[i] = cscale(w[i], inv);
}

}  // namespace

// One-sided Jacobi SVD of nprob blocks W[prob] (c rows of length n, i.e. the
// columns of S as rows).  W is overwritten by U*Sigma (rows).  Outputs:
// sigma (nprob x c, descending), order (nprob x c), kept (nprob), and
// Qt[prob] (kept x n rows, orthonormal).  ws: >= 64 bytes of device scratch.
// Returns the number of sweeps in *sweeps_out (device int).
CIRR_API int cirr_orth(cplx* W, long long ldw, long long wstride, int n, int c, int nprob, double rel_tol,
                       double* sigma, int* order, int* kept, cplx* Qt, long long ldq, long long qstride,
                       void* ws, int* sweeps_out, cudaStream_t stream) {
  if (n <= 0 || c <= 0 || nprob <= 0 || ldw < n || ldq < n) return CIRR_EINVAL;
  unsigned* bar = reinterpret_cast<unsigned*>(ws);
  int* counters = reinterpret_cast<int*>(bar + 2);
  cudaError_t e = cudaMemsetAsync(ws, 0, 64, stream);
  if (e != cudaSuccess) return (int)e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hestenes_kernel, HT, 0);
  const int cp = c + (c & 1);
  long long items = (long long)nprob * (cp / 2);
  int grid = (int)(items < (long long)sms * per_sm ? items : (long long)sms * per_sm);
  if (grid < 1) grid = 1;
  if (c > 1) {
    // rotation threshold on |x^H y| / (|x||y|): 16 sqrt(n) eps keeps it above the
    // rounding noise of an n-term dot product (sqrt(n) eps alone never converges)
    double tol = 16.0 * sqrt((double)n) * 1.1102230246251565e-16;
    int max_sweeps = 40;
    void* args[] = {&W, &ldw, &wstride, &n, &c, &nprob, &bar, &counters, &max_sweeps, &tol, &sweeps_out};
    e = cudaLaunchCooperativeKernel((void*)hestenes_kernel, dim3(grid), dim3(HT), args, 0, stream);
    cirr_note_launch();
    if (e != cudaSuccess) return (int)e;
  } else {
    e = cudaMemsetAsync(sweeps_out, 0, sizeof(int), stream);
    if (e != cudaSuccess) return (int)e;
  }
  size_t sm = sizeof(double) * (size_t)c;
  svd_finalize_kernel<<<nprob, 1024, sm, stream>>>(W, ldw, wstride, n, c, rel_tol, sigma, order, kept);
  CIRR_CHECK_LAUNCH();
  dim3 gq((n + 255) / 256 < 64 ? (n + 255) / 256 : 64, c, nprob);
  build_q_kernel<<<gq, 256, 0, stream>>>(W, ldw, wstride, n, c, sigma, order, kept, Qt, ldq, qstride);
  CIRR_CHECK_LAUNCH();
  return 0;
}
