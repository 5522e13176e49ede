// C-ABI for the batched DMMA GEMM (see gemm.cuh).
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

// Number of kernels launched by this library since load (host counter).
CIRR_API long long cirr_launch_count(void) { return __atomic_load_n(&g_cirr_launches, __ATOMIC_RELAXED); }

// 100 = the cubins in this library target sm_100a (B200).
CIRR_API int cirr_target_sm(void) { return 100; }
