// Ozaki-split complex128 GEMM update on the int8 tensor cores (ozaki.cu).
#pragma once
#include "common.cuh"

namespace cirr {
// true when the dense LU's k = 512 trailing updates take the int8 path (cirr_set_lu_gemm)
bool ozaki_enabled();
// shapes the int8 path takes: K a multiple of 32 (K' = 2K bytes in 64-byte stages)
bool ozaki_shape_ok(int M, int N, int K);
// slice workspace for one batch entry (bytes)
long long ozaki_ws_bytes_per_entry(int M, int N, int K);
// C -= A B, batch independent complex128 problems (row-major, strides in elements)
int ozaki_zgemm_sub(const cplx* A, long long lda, long long sA, const cplx* B, long long ldb, long long sB, cplx* C,
                    long long ldc, long long sC, int M, int N, int K, int batch, cudaStream_t stream);
// Factor slices for the solves (see ozaki.cu): bytes of the caller-owned cache
// (0: shape not taken), the split + registration, the release, and the cached
// trailing update (-1: no slices for this factor, take the DMMA path).
long long ozaki_factor_bytes(int n, int nfac);
int ozaki_split_factors(const cplx* LU, int n, long long ld, long long pstride, int nfac, void* cache,
                        cudaStream_t stream);
int ozaki_release(const cplx* LU);
void ozaki_invalidate(const void* p, long long bytes);
int ozaki_cached_update(const cplx* LU, int n, int col0, int kw, int a_row0, int M, const cplx* B, long long ldb,
                        long long sB, cplx* C, long long ldc, long long sC, int N, int batch, const int* pmap,
                        cudaStream_t stream);
}  // namespace cirr
