/* libcirr -- C ABI of the B200-native CIRR contour-integral stage.
 *
 * The reference (cieig, pure Python) has no FFI for this path; its plugin
 * surface is the Python call cirr_solve / solve_multi
 * (/root/reference/pkg/src/cieig/solvers.py:165-227, 312-339).  Each entry
 * below replaces one reference call site, cited per function; the Python
 * package paper_2511_01927_b200 binds them with ctypes (_lib.py) and keeps
 * the reference's Python signatures above them.
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer (PyTorch-owned buffers); complex
 *     values are complex128 interleaved (re, im) -- `cplx` = double2.
 *   - Matrices are row-major; `ld*` are leading dimensions and `s*`/`*stride`
 *     batch strides, in ELEMENTS.
 *   - Return 0 on success, a cudaError_t (> 0) on a CUDA error, or
 *     CIRR_EINVAL (100000) for invalid arguments.  No entry allocates device
 *     memory or synchronises the stream.
 *   - All work is enqueued on `stream`; results are deterministic
 *     (fixed-order reductions, no floating-point atomics).
 */
#ifndef CIRR_H
#define CIRR_H

#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double2 cirr_cplx;

#define CIRR_EINVAL 100000

/* K1 -- replaces linalg.py:62-63 (z*B - A and the max|M_ij| scale).
 * pencils[j] = z[j]*B - A (bitwise equal to numpy), maxabs[j] = max |.|. */
int cirr_assemble(const double* A, const double* B, int n, long long lda,
                  const cirr_cplx* z, int nz, cirr_cplx* pencils, long long ldp,
                  long long pencil_stride, double* maxabs, cudaStream_t stream);
/* cirr_assemble for pencils of many GEPs in one launch: pencil j uses the real
 * A, B at device addresses a_ptrs[j], b_ptrs[j] (device int64[nz]); bitwise
 * equal to cirr_assemble (solve_multi_batch's per-GEP linalg.py:62-63). */
int cirr_assemble_ptrs(const long long* a_ptrs, const long long* b_ptrs, int n, long long lda,
                       const cirr_cplx* z, int nz, cirr_cplx* pencils, long long ldp, long long pencil_stride,
                       double* maxabs, cudaStream_t stream);
/* Complex-valued A and B (complex128, row-major, ld lda): pencils[j] = z[j] B - A
 * with numpy's complex arithmetic (the reference's MatrixPencil carries complex
 * CSR values, sparse.py:14-43); maxabs as cirr_assemble. */
int cirr_assemble_c(const cirr_cplx* A, const cirr_cplx* B, int n, long long lda, const cirr_cplx* z, int nz,
                    cirr_cplx* pencils, long long ldp, long long pencil_stride, double* maxabs,
                    cudaStream_t stream);
/* out[0] = max |A - A^H|, out[1] = max |A| of a complex128 matrix (sparse.py:83-87). */
int cirr_hermitian_c(const cirr_cplx* A, int n, long long lda, double* out, cudaStream_t stream);

/* sparse.py:83-87 (is_hermitian) for real A: out[0] = max|A - A^T|, out[1] = max|A|. */
int cirr_symmetry(const double* A, int n, long long lda, double* out, cudaStream_t stream);

/* K2 -- replaces linalg.py:65-70 (splu + the 1e-14 pivot test inputs).
 * In-place P M = L U of `batch` pencils; ipiv/perm: batch x n int32;
 * minpiv[j] = min_i |U_ii|; info[j] = first exact zero pivot (1-based) or 0. */
int cirr_zgetrf_batched(cirr_cplx* pencils, int n, long long ld, long long pencil_stride,
                        int batch, int* ipiv, int* perm, double* minpiv, int* info, void* ws,
                        cudaStream_t stream);
/* Banded pencils (the stencil configs 1/2/3/5, stored dense): the same LU on
 * the band only -- panel rows stop at k+jb+kl, interchanges and U blocks at
 * column k+jb+kl+ku (fill-in bound), trailing updates cover kl x (kl+ku).  The
 * skipped entries are exact zeros, so the factors are bitwise those of
 * cirr_zgetrf_batched.  lbw: batch ints (zeroed by the caller) raised to L's
 * final lower bandwidth when interchanges move L entries beyond kl. */
int cirr_zgetrf_band(cirr_cplx* pencils, int n, long long ld, long long pencil_stride, int batch, int kl, int ku,
                     int* ipiv, int* perm, double* minpiv, int* info, int* lbw, void* ws, cudaStream_t stream);
/* out[0] = max(i-j), out[1] = max(j-i) over the nonzeros of an n x n real
 * (is_complex 0) or complex128 matrix, raised with atomicMax (zero out first;
 * one call per matrix gives the union of A's and B's patterns). */
int cirr_bandwidth(const void* M, int is_complex, int n, long long ld, int* out, cudaStream_t stream);
/* cirr_bandwidth for count (<= 65535) matrices at device addresses ptrs[i]
 * (device int64[count]), one launch: out[2i], out[2i+1] (zeroed first). */
int cirr_bandwidth_ptrs(const long long* ptrs, int count, int is_complex, int n, long long ld, int* out,
                        cudaStream_t stream);
/* ws bytes for cirr_zgetrf_batched (L11^-1 blocks; ws may be NULL: slower TRSM path) */
long long cirr_zgetrf_ws_bytes(int n, int batch);

/* K3a -- replaces linalg.py:46-52 (SuperLU gstrs) as used at solvers.py:124.
 * Y[j] = M_j^{-1} R[rhs_of[j]] (rhs_of: device int32[batch]). */
int cirr_zgetrs_batched(const cirr_cplx* LU, int n, long long ld, long long pencil_stride,
                        int batch, const int* perm, const cirr_cplx* R, long long ldr,
                        long long rstride, const int* rhs_of, int K, cirr_cplx* Y,
                        long long ldy, long long ystride, const cirr_cplx* Dinv, cudaStream_t stream);
/* The same solves for any subset of the nfac factors at LU: batch entry j uses
 * factor pencil_of[j] (device int32[batch]); perm and Dinv are indexed by
 * factor, rhs_of and Y by entry.  Lets contours that are not adjacent in the
 * factor buffer (refinement passes of a multi-pencil batch) share one call. */
int cirr_zgetrs_gather(const cirr_cplx* LU, int n, long long ld, long long pencil_stride, int nfac,
                       const int* pencil_of, int batch, const int* perm, const cirr_cplx* R, long long ldr,
                       long long rstride, const int* rhs_of, int K, cirr_cplx* Y, long long ldy,
                       long long ystride, const cirr_cplx* Dinv, cudaStream_t stream);
/* Inverses of the 128x128 diagonal blocks of L and U (optional input of
 * cirr_zgetrs_batched: the diagonal solves become TMA/DMMA GEMMs). */
long long cirr_diag_inv_bytes(int n, int batch);
int cirr_diag_inverses(const cirr_cplx* LU, int n, long long ld, long long pencil_stride, int batch,
                       cirr_cplx* Dinv, cudaStream_t stream);
/* 1 when cirr_zgetrs_batched reads Dinv for an n x K solve (K <= 2, or K > 16),
 * 0 when it does not (callers may then skip cirr_diag_inverses). */
int cirr_zgetrs_uses_dinv(int n, int K);

/* Engine plumbing (no reference counterpart): the batched GEMM with a
 * per-entry A operand at device address a_ptrs[b] (products with the pencils
 * of many GEPs without stacking them), a one-launch assembly of npiece device
 * blocks into a batched buffer (desc: device int64[8*npiece] =
 * {src address, src ld, rows, cols, dst entry, dst column, conj, dst ld or 0}), and a
 * stream-ordered zero fill.  Together they keep PyTorch to allocation only. */
int cirr_gemm_ptrs(int a_kind, int M, int N, int K, int batch, const long long* a_ptrs, long long lda,
                   const cirr_cplx* B, long long ldb, long long sB, cirr_cplx* C, long long ldc, long long sC,
                   double alpha, int beta, cudaStream_t stream);
int cirr_gather_blocks(int npiece, const long long* desc, long long max_elems, cirr_cplx* dst, long long ldd,
                       long long sd, cudaStream_t stream);
int cirr_zero(void* p, long long bytes, cudaStream_t stream);

/* K3a+K3b fused -- replaces solvers.py:121-129 as one call: the solves of
 * cirr_zgetrs_gather (pencil_of NULL: entry j uses factor j, as
 * cirr_zgetrs_batched) with the moment accumulation of cirr_moments (same
 * coef/off/St layout, M <= 16) done inside the solve, block row by block row
 * as the backward substitution finishes each one (L2-resident). */
int cirr_zgetrs_moments(const cirr_cplx* LU, int n, long long ld, long long pencil_stride, int nfac,
                        const int* pencil_of, int batch, const int* perm, const cirr_cplx* R, long long ldr,
                        long long rstride, const int* rhs_of, int K, cirr_cplx* Y, long long ldy,
                        long long ystride, const cirr_cplx* Dinv, const cirr_cplx* coef, int M, const int* off,
                        int n_sets, cirr_cplx* St, long long ld_st, long long sstride, cudaStream_t stream);

/* cirr_zgetrs_moments / _gather / _batched in one entry, cut to the factors'
 * bandwidths klL (L below the diagonal: max(kl, lbw of cirr_zgetrf_band)) and
 * kuU (U above: kl + ku); -1 = dense.  pencil_of NULL: entry j uses factor j;
 * coef NULL: no moment accumulation.  Bitwise equal to the dense entries. */
int cirr_zgetrs_band(const cirr_cplx* LU, int n, long long ld, long long pencil_stride, int nfac,
                     const int* pencil_of, int batch, const int* perm, const cirr_cplx* R, long long ldr,
                     long long rstride, const int* rhs_of, int K, cirr_cplx* Y, long long ldy, long long ystride,
                     const cirr_cplx* Dinv, const cirr_cplx* coef, int M, const int* off, int n_sets,
                     cirr_cplx* St, long long ld_st, long long sstride, int klL, int kuU, cudaStream_t stream);

/* K3b -- replaces solvers.py:121-129 (acc[m] += w_j zeta_j^m Y_j).
 * St[c] ((M*K) x n): row m*K+col = column col of S_m of contour c, summed over
 * pencils off[c]..off[c+1]-1 in order with coef[j*M+m]. */
int cirr_moments(const cirr_cplx* Y, long long ldy, long long ystride, int n, int K,
                 const cirr_cplx* coef, int M, const int* off, int n_sets, cirr_cplx* St,
                 long long ld_st, long long sstride, cudaStream_t stream);

/* K4 -- replaces linalg.py:107-119 (thin SVD + sigma >= rel_tol*sigma_max).
 * Householder QR of S + one-sided Jacobi SVD of R; W (c x n per problem: the
 * columns of S as rows) is overwritten; sigma/order: nprob x c (descending),
 * kept: nprob, Qt: kept x n rows (orthonormal columns of Q).
 * ws: cirr_orth_ws_bytes(c, nprob) bytes; *sweeps_out (device int). */
long long cirr_orth_ws_bytes(int c, int nprob);
int cirr_orth(cirr_cplx* W, long long ldw, long long wstride, int n, int c, int nprob,
              double rel_tol, double* sigma, int* order, int* kept, cirr_cplx* Qt,
              long long ldq, long long qstride, void* ws, int* sweeps_out, cudaStream_t stream);

/* FEAST basis -- replaces linalg.py:79-104 (orthonormalize, MGS x2 with drop_tol):
 * CGS2 per problem on the rows of Y (c x n); Qt[p] gets kept[p] orthonormal rows. */
int cirr_orthonormalize(const cirr_cplx* Y, long long ldy, long long sy, int n, int c, int nprob, double drop_tol,
                        cirr_cplx* Qt, long long ldq, long long sq, int* kept, cudaStream_t stream);

/* K5/K7 GEMM -- replaces sparse.py:98-103 (sparse_matmat for B V, A Q, B Q,
 * A X, B X) and the dense products of solvers.py:153-158.
 * C = beta*C + alpha*op(A)@B; a_kind 0: A complex, 1: conj(A), 2: A real f64. */
int cirr_gemm(int a_kind, int M, int N, int K, int batch, const void* A, long long lda,
              long long sA, const cirr_cplx* B, long long ldb, long long sB, cirr_cplx* C,
              long long ldc, long long sC, double alpha, int beta, cudaStream_t stream);

/* K6 -- replaces linalg.py:122-145 (dense_hermitian_gep) and adds the
 * non-Hermitian Rayleigh-Ritz (SURVEY.md 8(c) delta 3). */
long long cirr_small_eig_ws_bytes(int kmax);
int cirr_small_eig(int hermitian, const cirr_cplx* At, const cirr_cplx* Bt, long long ldin,
                   long long sin_, const int* kdim, int kmax, int nprob, void* ws, cirr_cplx* lam,
                   cirr_cplx* S, long long lds, long long sS, int* info, cudaStream_t stream);

/* K6 non-Hermitian (k <= 256): phase 1 eigenvalues (sorted by re, im) of
 * B~^-1 A~ via batched LU/solve, cooperative Hessenberg reduction and an
 * eigenvalue-only QR; phase 2 unit-norm eigenvectors for selected sorted
 * indices by inverse iteration + Householder back-transform.  Bt = NULL:
 * B~ = I (no LU). */
long long cirr_gen_eig_ws_bytes(int kmax, int nprob);
long long cirr_gen_eig_vec_scratch_bytes(int kmax, int nprob, int smax);
int cirr_gen_eig_values(const cirr_cplx* At, const cirr_cplx* Bt, const int* kdim, int kmax, int nprob, void* ws,
                        cirr_cplx* lam, int* info, cudaStream_t stream);
/* As cirr_gen_eig_values, with shift hints for the QR iteration: hint[p]
 * (ld hint_ld) holds hint_cnt[p] <= 256 approximate eigenvalues, e.g. the
 * previous refinement round's; when the Wilkinson shift lies within 5 % of an
 * unused hint the hint is the shift.  Same eigenvalues to rounding, fewer sweeps. */
int cirr_gen_eig_values_hinted(const cirr_cplx* At, const cirr_cplx* Bt, const int* kdim, int kmax, int nprob,
                               void* ws, cirr_cplx* lam, int* info, const cirr_cplx* hint, const int* hint_cnt,
                               int hint_ld, cudaStream_t stream);
int cirr_gen_eig_vectors(void* ws, const int* kdim, int kmax, int nprob, const cirr_cplx* lam, const int* sel,
                         const int* sel_cnt, int smax, void* scratch, cirr_cplx* S, long long lds, long long sS,
                         cudaStream_t stream);

/* K6 non-Hermitian, refinement rounds (solvers.py:200-205 feeding 187-198):
 * eigenpairs of (A~, B~) from approximate eigenvectors, by Newton refinement of
 * the eigenbasis on batched DMMA GEMMs and the batched LU/solve instead of the
 * sequential Hessenberg QR.  W0h[p] (ld ldw, stride sw) = W0^H, e.g. S^H Q for
 * the refinement block S and its orthonormal basis Q.  lam, S as
 * cirr_gen_eig_values / cirr_gen_eig_vectors (sorted by (re, im); unit-norm
 * eigenvectors in that order, all k of them); info: 0 ok, -1 not converged
 * within max_iter steps or B~ W0 singular (the caller then uses the
 * QR path for that problem).  ws: cirr_gen_eig_refine_ws_bytes(kmax, nprob). */
long long cirr_gen_eig_refine_ws_bytes(int kmax, int nprob);
int cirr_gen_eig_refine(const cirr_cplx* At, const cirr_cplx* Bt, const int* kdim, int kmax, int nprob,
                        const cirr_cplx* W0h, long long ldw, long long sw, int max_iter, void* ws, cirr_cplx* lam,
                        cirr_cplx* S, long long lds, long long sS, int* info, cudaStream_t stream);

/* Certified CholeskyQR2 basis (the fast path of cirr_orth for full-rank blocks):
 * W[p] (c x n rows = the columns of S, cdim[p] valid) -> Qt[p] (cdim[p]
 * orthonormal rows spanning range(S), zero rows after); ok[p] = 1 when
 * ||R||_F ||R^-1||_F <= kappa_max (full rank certified), else 0 and the caller
 * uses cirr_orth.  Replaces linalg.py:107-119 when no singular value is cut.
 * ws: cirr_orth_cholqr2_ws_bytes(n, c, nprob). */
long long cirr_orth_cholqr2_ws_bytes(int n, int c, int nprob);
int cirr_orth_cholqr2(const cirr_cplx* W, long long ldw, long long wstride, int n, int c, int nprob,
                      const int* cdim, double kappa_max, cirr_cplx* Qt, long long ldq, long long qstride,
                      void* ws, int* ok, cudaStream_t stream);

/* debug: clock64 marks of the last cirr_orth launch (4 entries) */
int cirr_orth_phases(long long* host_out);

/* debug: of the last cirr_gen_eig_refine, the step at which problems 0..7
 * converged (-1: not) and the columns the block step replaced (16 ints, host) */
int cirr_gen_eig_refine_stats(int* host_out);

/* debug: sweeps, rotations and clock64 cycles of the last eigenvalue-QR launch (8 entries) */
int cirr_gen_eig_qr_stats(long long* host_out);

/* debug: clock64 stamps of the phases of the last general-eig launch (problem 0), 10 entries (host buffer) */
int cirr_small_eig_phases(long long* host_out);

/* K7 -- replaces solvers.py:140-147 (_residuals). */
int cirr_residuals(const cirr_cplx* AX, const cirr_cplx* BX, long long ld, long long stride, int n,
                   const cirr_cplx* lam, long long lstride, const int* kdim, int kmax, int nprob,
                   double* res, long long rstride, cudaStream_t stream);

/* solvers.py:196 (xs[:, keep]) */
int cirr_gather_cols(const cirr_cplx* in, long long ldi, long long si, const int* idx, long long sidx,
                     const int* cnt, int cmax, int n, int nprob, cirr_cplx* out, long long ldo,
                     long long so, cudaStream_t stream);

/* out[b][r][c] = op(in[src[b]][r][col0[b] + c]), op = conj when cj[b] (conjugate-pair variant) */
int cirr_copy_cols(const cirr_cplx* in, long long ldi, long long si, const int* src, const int* col0,
                   const int* cj, int n, int K, int count, cirr_cplx* out, long long ldo, long long so,
                   cudaStream_t stream);

/* layout helper: out[b] = in[b]^T (or ^H when conj != 0) */
int cirr_transpose(int conj, const cirr_cplx* in, long long ldi, long long si, int rows, int cols,
                   int batch, cirr_cplx* out, long long ldo, long long so, cudaStream_t stream);

/* KDE sparsity upstream of the solve (kernels.py:38-67 kde_eval, used by
 * contours.py:175-192): out[i] = sum_j exp(-coef (ts[i] - eigs[j])^2), summed in
 * j order.  ts (nt), eigs (ne), out (nt): device float64. */
int cirr_kde_eval(const double* ts, int nt, const double* eigs, int ne, double coef, double* out,
                  cudaStream_t stream);

/* Int8 tensor-core path of the k = 512 trailing updates of K2 (no reference
 * counterpart; the reference factors with SuperLU in FP64, linalg.py:55-71):
 * C -= A B for `batch` complex128 problems (row-major, strides in elements) by
 * the Ozaki splitting -- rows of A and columns of B scaled by powers of two and
 * cut into eight signed 7-bit digits, the 36 digit products exact in int32 on
 * tcgen05.mma kind::i8, recombined in integers and converted once to FP64.
 * K must be a multiple of 32.  Error per k-term below 2^-53 rowmax(A) colmax(B). */
int cirr_ozaki_zgemm_sub(const cirr_cplx* A, long long lda, long long sA, const cirr_cplx* B, long long ldb,
                         long long sB, cirr_cplx* C, long long ldc, long long sC, int M, int N, int K, int batch,
                         cudaStream_t stream);

/* Int8 path of the blocked solves (K3): the factors are constant over the
 * solve passes of a run (solvers.py:113-130 applies the same LU every pass), so
 * their digit slices are cut once after cirr_zgetrf_batched into a caller-owned
 * buffer of cirr_ozaki_factor_bytes(n, nfac) bytes (0: shape not taken -- n
 * must be a multiple of 512, at least 1024) and registered under the LU
 * address; the k = 512 trailing updates of every later cirr_zgetrs_* call on
 * those factors (any sub-range of them, dense bandwidths) then run on the int8
 * tensor cores.  Release before the factors or the buffer are freed or
 * refactored. */
long long cirr_ozaki_factor_bytes(int n, int nfac);
int cirr_ozaki_split_factors(const cirr_cplx* LU, int n, long long ld, long long pencil_stride, int nfac,
                             void* cache, cudaStream_t stream);
int cirr_ozaki_release(const cirr_cplx* LU);

/* Arithmetic of the dense LU's k = 512 trailing updates (K2): 0 = FP64 DMMA
 * (zgemm_sub_tma), 1 = the int8 tensor-core path above.  Banded pencils and the
 * in-step updates always take DMMA.  Returns the previous mode; any other
 * argument only queries.  Default 1; CIRR_LU_GEMM=dmma starts in mode 0. */
int cirr_set_lu_gemm(int mode);

/* number of kernels this library has launched since it was loaded (host counter) */
long long cirr_launch_count(void);

/* library identification: compute capability the cubins target (100 = sm_100a) */
int cirr_target_sm(void);

/* Concurrency: cap the CTAs of the cooperative latency-bound kernels (K4 orth,
 * Hessenberg) so they can run beside the bulk GEMMs of another stream
 * (0 = whole GPU, the default).  Returns the previous cap. */
int cirr_set_coop_ctas(int ctas);

/* Concurrency: cap the CTAs of the persistent TMA GEMM (LU trailing updates and
 * blocked solves) so latency-bound kernels of another stream find free SMs
 * (0 = every SM, the default).  Returns the previous cap. */
int cirr_set_gemm_ctas(int ctas);

/* Memory: callback run when a stream-ordered scratch allocation (split-K
 * partials, look-back flags, WY workspaces) fails because another allocator
 * holds the free HBM -- the Python host passes a function that empties
 * PyTorch's cache; the allocation is then retried once.  NULL clears it. */
void cirr_set_oom_handler(void (*fn)(void));

#ifdef __cplusplus
}
#endif
#endif /* CIRR_H */
