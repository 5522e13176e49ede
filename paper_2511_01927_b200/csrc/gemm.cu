// C-ABI for the batched DMMA GEMM (see gemm.cuh).
#include <mutex>
#include <utility>
#include <vector>
#include "gemm.cuh"

using namespace cirr;

namespace {
__global__ void zero_kernel(cplx* C, int M, int N, long long ldc, long long sC) {
  const int b = blockIdx.z;
  const int r = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < M && c < N) C[(long long)b * sC + (long long)r * ldc + c] = cmk(0.0, 0.0);
}
}  // namespace

// a_kind: 0 = A complex, 1 = conj(A) complex, 2 = A real float64.
// C[b] = beta*C[b] + alpha * op(A[b]) @ B[b]; all row-major; strides in elements.
CIRR_API int cirr_gemm(int a_kind, int M, int N, int K, int batch,
                       const void* A, long long lda, long long sA,
                       const cplx* B, long long ldb, long long sB,
                       cplx* C, long long ldc, long long sC,
                       double alpha, int beta, cudaStream_t stream) {
  if (M < 0 || N < 0 || K < 0 || batch < 0 || a_kind < 0 || a_kind > 2) return CIRR_EINVAL;
  if (M == 0 || N == 0 || batch == 0) return 0;
  if (K == 0) {
    if (beta) return 0;
    dim3 grid((N + 127) / 128, M, batch);
    zero_kernel<<<grid, 128, 0, stream>>>(C, M, N, ldc, sC);
    CIRR_CHECK_LAUNCH();
    return 0;
  }
  GemmArgs g{M, N, K, batch, A, lda, sA, B, ldb, sB, C, ldc, sC, alpha, beta};
  switch (a_kind) {
    case 0: return gemm_launch<false, false>(g, stream);
    case 1: return gemm_launch<false, true>(g, stream);
    default: return gemm_launch<true, false>(g, stream);
  }
}

// cirr_gemm with a per-entry A operand: A of batch entry b is the matrix at
// device address a_ptrs[b] (device int64[batch]), so products with the
// pencils of many GEPs (solve_multi_batch) need no stacked copy of A and B.
CIRR_API int cirr_gemm_ptrs(int a_kind, int M, int N, int K, int batch, const long long* a_ptrs, long long lda,
                            const cplx* B, long long ldb, long long sB, cplx* C, long long ldc, long long sC,
                            double alpha, int beta, cudaStream_t stream) {
  if (M < 0 || N < 0 || K <= 0 || batch < 0 || a_kind < 0 || a_kind > 2 || a_ptrs == nullptr) return CIRR_EINVAL;
  if (M == 0 || N == 0 || batch == 0) return 0;
  GemmArgs g{M, N, K, batch, nullptr, lda, 0, B, ldb, sB, C, ldc, sC, alpha, beta};
  g.a_ptrs = a_ptrs;
  switch (a_kind) {
    case 0: return gemm_launch<false, false>(g, stream);
    case 1: return gemm_launch<false, true>(g, stream);
    default: return gemm_launch<true, false>(g, stream);
  }
}

namespace {
// One complex block per piece: dst[d][r][c0 + c] = op(src[r * ld + c]) for
// r < rows, c < cols (op = conj when flagged).  Piece descriptors (int64):
// {src address, src ld, rows, cols, d, c0, conj, dst ld (0: ldd)}.
__global__ void gather_blocks_kernel(const long long* __restrict__ desc, cplx* __restrict__ dst, long long ldd,
                                     long long sd) {
  const long long* q = desc + 8LL * blockIdx.y;
  const cplx* src = reinterpret_cast<const cplx*>(q[0]);
  const long long ld = q[1];
  const int rows = (int)q[2], cols = (int)q[3];
  cplx* out = dst + q[4] * sd + q[5];
  const bool cj = q[6] != 0;
  if (q[7] > 0) ldd = q[7];
  const long long total = (long long)rows * cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / cols), c = (int)(e % cols);
    cplx v = src[r * ld + c];
    if (cj) v.y = -v.y;
    out[r * ldd + c] = v;
  }
}
}  // namespace

// Assemble npiece device blocks (any addresses and leading dimensions) into
// one batched buffer in one launch: the padded right-hand-side, moment and
// basis stacks of the engine.  desc: device int64[7 * npiece] (see above);
// max_elems: the largest rows * cols over the pieces.  Padding is not
// written: zero it first (cirr_zero) where it matters.
CIRR_API int cirr_gather_blocks(int npiece, const long long* desc, long long max_elems, cplx* dst, long long ldd,
                                long long sd, cudaStream_t stream) {
  if (npiece < 0 || max_elems < 0) return CIRR_EINVAL;
  if (npiece == 0 || max_elems == 0) return 0;
  long long bx = (max_elems + 255) / 256;
  if (bx > 1024) bx = 1024;
  dim3 grid((unsigned)bx, (unsigned)npiece);
  gather_blocks_kernel<<<grid, 256, 0, stream>>>(desc, dst, ldd, sd);
  CIRR_CHECK_LAUNCH();
  return 0;
}

// bytes of device memory set to zero, stream-ordered (a memset, not a kernel).
CIRR_API int cirr_zero(void* p, long long bytes, cudaStream_t stream) {
  if (bytes <= 0) return 0;
  return (int)cudaMemsetAsync(p, 0, (size_t)bytes, stream);
}

long long g_cirr_launches = 0;
int g_cirr_coop_cap = 0;
int g_cirr_gemm_cap = 0;

// The persistent TMA GEMM uses at most `ctas` CTAs when > 0 (SMs left free for
// the latency-bound kernels of another stream).  Returns the old cap.
CIRR_API int cirr_set_gemm_ctas(int ctas) {
  const int old = g_cirr_gemm_cap;
  g_cirr_gemm_cap = ctas > 0 ? ctas : 0;
  return old;
}

// Cooperative kernels (K4 orth, Hessenberg) use at most `ctas` CTAs when > 0,
// leaving the rest of the GPU to GEMMs on other streams.  Returns the old cap.
CIRR_API int cirr_set_coop_ctas(int ctas) {
  const int old = g_cirr_coop_cap;
  g_cirr_coop_cap = ctas > 0 ? ctas : 0;
  return old;
}

namespace {
constexpr int kCtrSlots = 256;
struct CtrPool {
  int dev;
  int* base;
  std::vector<cudaStream_t> streams;
};
std::mutex g_ctr_mu;
std::vector<CtrPool> g_ctr;
}  // namespace

// One {next tile, finished CTAs} pair per (device, stream).  The pool is
// allocated and zeroed synchronously on first use (before any concurrent
// launch), and each kernel leaves its pair at zero when it exits.
int* cirr_tile_counter(cudaStream_t stream) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_ctr_mu);
  CtrPool* pool = nullptr;
  for (auto& p : g_ctr)
    if (p.dev == dev) pool = &p;
  if (!pool) {
    int* base = nullptr;
    if (cudaMalloc(&base, 2 * sizeof(int) * kCtrSlots) != cudaSuccess) return nullptr;
    if (cudaMemset(base, 0, 2 * sizeof(int) * kCtrSlots) != cudaSuccess) return nullptr;
    if (cudaDeviceSynchronize() != cudaSuccess) return nullptr;
    g_ctr.push_back(CtrPool{dev, base, {}});
    pool = &g_ctr.back();
  }
  for (size_t i = 0; i < pool->streams.size(); ++i)
    if (pool->streams[i] == stream) return pool->base + 2 * i;
  if ((int)pool->streams.size() >= kCtrSlots) return nullptr;
  pool->streams.push_back(stream);
  return pool->base + 2 * (pool->streams.size() - 1);
}

namespace {
void (*g_oom_handler)(void) = nullptr;
}

CIRR_API void cirr_set_oom_handler(void (*fn)(void)) { g_oom_handler = fn; }

cudaError_t cirr_malloc_async(void** p, size_t bytes, cudaStream_t stream) {
  cudaError_t e = cudaMallocAsync(p, bytes, stream);
  if (e == cudaErrorMemoryAllocation && g_oom_handler) {
    cudaGetLastError();  // clear the failed allocation's error
    g_oom_handler();
    e = cudaMallocAsync(p, bytes, stream);
  }
  return e;
}

// Number of kernels launched by this library since load (host counter).
CIRR_API long long cirr_launch_count(void) { return __atomic_load_n(&g_cirr_launches, __ATOMIC_RELAXED); }

// 100 = the cubins in this library target sm_100a (B200).
CIRR_API int cirr_target_sm(void) { return 100; }
