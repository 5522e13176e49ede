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

// Number of kernels launched by this library since load (host counter).
CIRR_API long long cirr_launch_count(void) { return __atomic_load_n(&g_cirr_launches, __ATOMIC_RELAXED); }

// 100 = the cubins in this library target sm_100a (B200).
CIRR_API int cirr_target_sm(void) { return 100; }
