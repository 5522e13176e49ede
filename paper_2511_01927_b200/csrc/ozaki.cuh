// Ozaki-split complex128 GEMM update on the int8 tensor cores (ozaki.cu).
#pragma once
#include "common.cuh"

namespace cirr {
// shapes the int8 path takes: K a multiple of 32 (K' = 2K bytes in 64-byte stages)
bool ozaki_shape_ok(int M, int N, int K);
// slice workspace for one batch entry (bytes)
long long ozaki_ws_bytes_per_entry(int M, int N, int K);
// C -= A B, batch independent complex128 problems (row-major, strides in elements)
int ozaki_zgemm_sub(const cplx* A, long long lda, long long sA, const cplx* B, long long ldb, long long sB, cplx* C,
                    long long ldc, long long sC, int M, int N, int K, int batch, cudaStream_t stream);
}  // namespace cirr
