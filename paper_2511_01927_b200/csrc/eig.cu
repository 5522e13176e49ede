// K6: the small projected eigenproblem, one CTA per contour.
//
// Replaces linalg.py:122-145 (dense_hermitian_gep: Cholesky test +
// scipy.linalg.eigh) as called from solvers.py:150-158, plus the
// non-Hermitian Rayleigh-Ritz the reference lacks (SURVEY.md 8(c) delta 3).
//
//  * herm_eig_kernel: symmetrise A~, B~ (solvers.py:155-156); Cholesky
//    B~ = L L^H (failure -> info > 0, raised as IndefiniteBError); A' =
//    L^-1 A~ L^-H; cyclic parallel Jacobi (circle-method rounds) on A';
//    s = L^-H W (B~-orthonormal); eigenvalues ascending.
//  * gen_eig_kernel: M = B~^-1 A~ (partial-pivot LU), Householder Hessenberg
//    reduction, single-shift complex QR (Wilkinson shift, exceptional shifts
//    at 10/20 iterations, zlahqr-style deflation) accumulating Z, eigenvectors
//    by back substitution on the Schur form, unit 2-norm; eigenvalues sorted
//    by (re, im) as numpy sorts complex values.
//
// k <= 1024.  Matrices live in a global workspace (L2 resident at these
// sizes); every reduction is fixed-order, so results are reproducible.
#include "common.cuh"
#include <cstdlib>

// herm_eig_kernel<SM, MODE>: the MODE 1 / 2 instances return before the
// Jacobi loops (reported as unreachable)
#pragma nv_diag_suppress 128

namespace {

constexpr int ET = 1024;
constexpr int GT = 256;         // threads of the general (non-Hermitian) solver
constexpr int QC = 16;          // rotations per chunk of a QR sweep
constexpr int WLD = QC + 4;     // window leading dimension

// phase timestamps of problem 0 (clock64), read back with cirr_small_eig_phases
__device__ long long g_eig_phase[16];
#define EIG_MARK(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_eig_phase[i] = clock64(); } while (0)
constexpr double EPS = 1.1102230246251565e-16;

struct EigWs {
  cplx* A;   // k x k
  cplx* L;   // k x k
  cplx* V;   // k x k
  cplx* T;   // k x k
  cplx* vec; // 4k
  double* d; // 4k
};

__device__ __forceinline__ EigWs carve(void* ws, long long wstride_bytes, int prob, int kmax) {
  unsigned char* base = reinterpret_cast<unsigned char*>(ws) + (long long)prob * wstride_bytes;
  EigWs w;
  const long long kk = (long long)kmax * kmax;
  w.A = reinterpret_cast<cplx*>(base);
  w.L = w.A + kk;
  w.V = w.L + kk;
  w.T = w.V + kk;
  w.vec = w.T + kk;
  w.d = reinterpret_cast<double*>(w.vec + 4 * (long long)kmax);
  return w;
}


// Element-wise read-modify-write over `total` items with U loads in flight per
// thread: all U loads of a batch are issued before any store, so L2 latency
// is paid once per batch instead of once per element (the compiler cannot
// reorder a load past a possibly-aliasing store on its own).
template <int U, typename AddrF, typename UpdF>
__device__ __forceinline__ void batched_rmw(int total, int nthreads, AddrF addr, UpdF upd) {
  for (int e0 = threadIdx.x; e0 < total; e0 += nthreads * U) {
    cplx* ptr[U];
    cplx val[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * nthreads;
      ptr[u] = e < total ? addr(e) : nullptr;
      if (ptr[u]) val[u] = *ptr[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ptr[u]) *ptr[u] = upd(e0 + u * nthreads, val[u]);
  }
}

__device__ __forceinline__ void jrot(double app, double aqq, cplx apq, double& cs, cplx& se) {
  // rotation J = [[c, s e^{i phi}], [-s e^{-i phi}, c]] zeroing apq of [[app, apq], [conj, aqq]]
  const double ag = cabs(apq);
  const double zeta = (aqq - app) / (2.0 * ag);
  const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  cs = 1.0 / sqrt(1.0 + t * t);
  const double sn = t * cs;
  se = cmk(sn * apq.x / ag, sn * apq.y / ag);
}

__device__ __forceinline__ void rr_pair(int round, int kk, int cp, int& p, int& q) {
  if (kk == 0) { p = cp - 1; q = round; }
  else { p = (round + kk) % (cp - 1); q = (round - kk + (cp - 1)) % (cp - 1); }
  if (p > q) { int t = p; p = q; q = t; }
}

// MODE 0: the whole solve (Jacobi on A' = L^-1 A~ L^-H in this CTA).
// MODE 1: stop after A' -- write it as the rows of W (W[j][i] = A'[i][j], the
//         column-as-row layout of cirr_orth) for the cooperative one-sided
//         Jacobi across the GPU, keep L and A'.
// MODE 2: finish from that SVD: A' HPD means its singular vectors are its
//         eigenvectors and sigma its eigenvalues; every pair is checked by its
//         Rayleigh quotient (an indefinite A' has lambda = -sigma somewhere),
//         and a failing problem gets info = -2 for a MODE 0 rerun.
// MODE 3: MODE 0 only for the problems MODE 2 flagged.
template <bool SM, int MODE = 0>
__global__ void __launch_bounds__(ET) herm_eig_kernel(const cplx* __restrict__ At, const cplx* __restrict__ Bt,
                                                      long long ldin, long long sin_, const int* __restrict__ kdim,
                                                      int kmax, void* ws, long long wstride,
                                                      cplx* __restrict__ lam, cplx* __restrict__ S, long long lds,
                                                      long long sS, int* __restrict__ info,
                                                      const cplx* __restrict__ Qt = nullptr,
                                                      const double* __restrict__ sigma = nullptr) {
  extern __shared__ __align__(16) cplx hsm[];   // A and V when they fit (in_smem)
  __shared__ double red[32];
  __shared__ double rot_c[512];
  __shared__ cplx rot_s[512];
  __shared__ int rot_p[512], rot_q[512];
  __shared__ int s_flag, s_count;
  const int prob = blockIdx.x;
  const int k = kdim[prob];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (MODE == 3 && info[prob] != -2) return;
  if (MODE == 2 && info[prob] != 0) return;   // Cholesky failure in MODE 1
  EigWs w = carve(ws, wstride, prob, kmax);
  const cplx* Ai = At + (long long)prob * sin_;
  const cplx* Bi = Bt + (long long)prob * sin_;
  cplx *A = w.A, *L = w.L, *V = w.V, *T = w.T;
  if (SM) {  // A, V in shared memory: every Jacobi round costs shared-memory latency, not an L2 round trip
    A = hsm;
    V = hsm + (long long)kmax * (kmax + 1);
  }
  const int ld = kmax;
  const int la = SM ? kmax + 1 : kmax;  // A / V row length (padded in shared memory: column walks hit distinct banks)
  if (tid == 0) s_flag = 0;
  if (MODE == 2) {
    // Rayleigh check and the eigenvectors from the SVD (Qt row r = u_r, sigma descending)
    __syncthreads();
    const cplx* Qp = Qt + (long long)prob * kmax * kmax;
    const double* sg = sigma + (long long)prob * kmax;
    const double smax = sg[0];
    // V[i][r] = u_r[i]; T[i][r] = (A' u_r)[i]
    for (int e = tid; e < k * k; e += ET) {
      const int i = e / k, r = e % k;
      V[i * ld + r] = Qp[(long long)r * kmax + i];
    }
    __syncthreads();
    for (int e = tid; e < k * k; e += ET) {
      const int i = e / k, r = e % k;
      cplx v = cmk(0.0, 0.0);
      for (int l = 0; l < k; ++l) cfma(v, A[i * ld + l], V[l * ld + r]);
      T[i * ld + r] = v;
    }
    __syncthreads();
    for (int r = wid; r < k; r += ET / 32) {
      double re = 0.0, pad = 0.0;
      for (int i = lane; i < kmax; i += 32) {
        if (i < k) re += cconjmul(V[i * ld + r], T[i * ld + r]).x;
        else pad += cabs2(Qp[(long long)r * kmax + i]);
      }
      re = warp_sum(re);
      pad = warp_sum(pad);
      if (lane == 0 && (!(fabs(re - sg[r]) <= 1e-10 * smax) || !(sg[r] > 1e-13 * smax) || pad > 1e-20)) s_flag = 1;
    }
    __syncthreads();
    if (s_flag) {
      if (tid == 0) info[prob] = -2;
      return;
    }
    // eigenvalues ascending: sigma is descending, so rank r -> k - 1 - r; s = L^-H u
    for (int r = tid; r < k; r += ET) lam[(long long)prob * kmax + (k - 1 - r)] = cmk(sg[r], 0.0);
    cplx* Sp = S + (long long)prob * sS;
    for (int c = tid; c < k; c += ET) {
      const int rank = k - 1 - c;
      for (int i = k - 1; i >= 0; --i) {
        cplx v = V[i * ld + c];
        for (int l = i + 1; l < k; ++l) cfms(v, cconj(L[l * ld + i]), T[l * ld + c]);
        v = cscale(v, 1.0 / L[i * ld + i].x);
        T[i * ld + c] = v;
        Sp[(long long)i * lds + rank] = v;
      }
    }
    return;
  }
  // 1. symmetrise
  for (int e = tid; e < k * k; e += ET) {
    int r = e / k, c = e % k;
    cplx a = Ai[(long long)r * ldin + c], at = Ai[(long long)c * ldin + r];
    cplx b = Bi[(long long)r * ldin + c], bt = Bi[(long long)c * ldin + r];
    A[r * la + c] = cmk(0.5 * (a.x + at.x), 0.5 * (a.y - at.y));
    L[r * ld + c] = cmk(0.5 * (b.x + bt.x), 0.5 * (b.y - bt.y));
  }
  __syncthreads();
  // 2. Cholesky (lower) of L in place
  for (int j = 0; j < k; ++j) {
    const double djj = L[j * ld + j].x;
    if (!(djj > 0.0)) {
      if (tid == 0) s_flag = j + 1;
      __syncthreads();
      break;
    }
    const double dj = sqrt(djj);
    __syncthreads();
    if (tid == 0) L[j * ld + j] = cmk(dj, 0.0);
    for (int r = j + 1 + tid; r < k; r += ET) L[r * ld + j] = cscale(L[r * ld + j], 1.0 / dj);
    __syncthreads();
    const int m = k - j - 1;
    for (int e = tid; e < m * m; e += ET) {
      int r = j + 1 + e / m, c = j + 1 + e % m;
      if (c <= r) cfms(L[r * ld + c], L[r * ld + j], cconj(L[c * ld + j]));
    }
    __syncthreads();
  }
  if (s_flag) {
    if (tid == 0) info[prob] = s_flag;
    return;
  }
  // 3. X = L^-1 A (column per thread), then A' = L^-1 X^H  (into T)
  for (int c = tid; c < k; c += ET) {
    for (int i = 0; i < k; ++i) {
      cplx v = A[i * la + c];
      for (int l = 0; l < i; ++l) cfms(v, L[i * ld + l], A[l * la + c]);
      A[i * la + c] = cscale(v, 1.0 / L[i * ld + i].x);
    }
  }
  __syncthreads();
  for (int c = tid; c < k; c += ET) {
    for (int i = 0; i < k; ++i) {
      cplx v = cconj(A[c * la + i]);
      for (int l = 0; l < i; ++l) cfms(v, L[i * ld + l], T[l * ld + c]);
      T[i * ld + c] = cscale(v, 1.0 / L[i * ld + i].x);
    }
  }
  __syncthreads();
  double fro = 0.0;
  for (int e = tid; e < k * k; e += ET) {
    int r = e / k, c = e % k;
    cplx a = T[r * ld + c], at = T[c * ld + r];
    cplx v = cmk(0.5 * (a.x + at.x), 0.5 * (a.y - at.y));
    A[r * la + c] = v;
    V[r * la + c] = cmk(r == c ? 1.0 : 0.0, 0.0);
    fro += cabs2(v);
  }
  fro = sqrt(block_sum(fro, red));
  __syncthreads();
  if (MODE == 1) {
    // A' for the cooperative SVD: W[j][i] = A'[i][j] (T), zero padded to kmax
    for (int e = tid; e < kmax * kmax; e += ET) {
      const int j = e / kmax, i = e % kmax;
      T[e] = (i < k && j < k) ? A[i * la + j] : cmk(0.0, 0.0);
    }
    if (tid == 0) info[prob] = 0;
    return;
  }
  // 4. parallel cyclic Jacobi
  const int cp = k + (k & 1), np = cp / 2;
  const double small = 1e-300 + 1e-18 * fro;
  for (int sweep = 0; sweep < 40 && k > 1; ++sweep) {
    if (tid == 0) s_count = 0;
    __syncthreads();
    for (int round = 0; round < cp - 1; ++round) {
      for (int t = tid; t < np; t += ET) {
        int p, q;
        rr_pair(round, t, cp, p, q);
        rot_p[t] = p; rot_q[t] = q; rot_c[t] = 1.0; rot_s[t] = cmk(0.0, 0.0);
        if (q < k) {
          const double app = A[p * la + p].x, aqq = A[q * la + q].x;
          const cplx apq = A[p * la + q];
          const double ag = cabs(apq);
          if (ag > small && ag > EPS * sqrt(fabs(app)) * sqrt(fabs(aqq))) {
            double cs; cplx se;
            jrot(app, aqq, apq, cs, se);
            rot_c[t] = cs; rot_s[t] = se;
            atomicAdd(&s_count, 1);
          } else {
            rot_q[t] = k;  // skip
          }
        }
      }
      __syncthreads();
      // columns: A <- A J, V <- V J (one warp per rotation, lanes over rows)
      for (int t = wid; t < np; t += ET / 32) {
        const int p = rot_p[t], q = rot_q[t];
        if (q >= k) continue;
        const double cs = rot_c[t];
        const cplx se = rot_s[t], sec = cconj(se);
        for (int r = lane; r < k; r += 32) {
          cplx x = A[r * la + p], y = A[r * la + q];
          A[r * la + p] = csub(cscale(x, cs), cmul(sec, y));
          A[r * la + q] = cadd(cmul(se, x), cscale(y, cs));
          x = V[r * la + p]; y = V[r * la + q];
          V[r * la + p] = csub(cscale(x, cs), cmul(sec, y));
          V[r * la + q] = cadd(cmul(se, x), cscale(y, cs));
        }
      }
      __syncthreads();
      // rows: A <- J^H A (one warp per rotation, lanes over columns)
      for (int t = wid; t < np; t += ET / 32) {
        const int p = rot_p[t], q = rot_q[t];
        if (q >= k) continue;
        const double cs = rot_c[t];
        const cplx se = rot_s[t], sec = cconj(se);
        for (int c = lane; c < k; c += 32) {
          cplx x = A[p * la + c], y = A[q * la + c];
          A[p * la + c] = csub(cscale(x, cs), cmul(se, y));
          A[q * la + c] = cadd(cmul(sec, x), cscale(y, cs));
        }
      }
      __syncthreads();
      for (int t = tid; t < np; t += ET) {
        const int p = rot_p[t], q = rot_q[t];
        if (q >= k) continue;
        A[p * la + q] = cmk(0.0, 0.0);
        A[q * la + p] = cmk(0.0, 0.0);
        A[p * la + p].y = 0.0;
        A[q * la + q].y = 0.0;
      }
      __syncthreads();
    }
    if (s_count == 0) break;
    __syncthreads();
  }
  // 5. sort ascending, s = L^-H W
  for (int i = tid; i < k; i += ET) {
    const double li = A[i * la + i].x;
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double lj = A[j * la + j].x;
      rank += (lj < li) || (lj == li && j < i);
    }
    w.d[i] = (double)rank;
    lam[(long long)prob * kmax + rank] = cmk(li, 0.0);
  }
  __syncthreads();
  cplx* Sp = S + (long long)prob * sS;
  for (int c = tid; c < k; c += ET) {
    const int rank = (int)w.d[c];
    for (int i = k - 1; i >= 0; --i) {
      cplx v = V[i * la + c];
      for (int l = i + 1; l < k; ++l) cfms(v, cconj(L[l * ld + i]), T[l * ld + c]);
      v = cscale(v, 1.0 / L[i * ld + i].x);
      T[i * ld + c] = v;
      Sp[(long long)i * lds + rank] = v;
    }
  }
  if (tid == 0) info[prob] = 0;
}

// --------------------------------------------------------------------------
// non-Hermitian

__device__ cplx csqrt_(cplx z) {
  const double r = cabs(z);
  if (r == 0.0) return cmk(0.0, 0.0);
  double x = sqrt(0.5 * (r + fabs(z.x)));
  double y = 0.5 * z.y / x;
  if (z.x >= 0.0) return cmk(x, y);
  return cmk(fabs(y), z.y >= 0.0 ? x : -x);
}

__global__ void __launch_bounds__(GT) gen_eig_kernel(const cplx* __restrict__ At, const cplx* __restrict__ Bt,
                                                     long long ldin, long long sin_, const int* __restrict__ kdim,
                                                     int kmax, void* ws, long long wstride,
                                                     cplx* __restrict__ lam, cplx* __restrict__ S, long long lds,
                                                     long long sS, int* __restrict__ info) {
  __shared__ double red[32];
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ int s_int[4];
  __shared__ cplx s_c[4];
  __shared__ cplx win[(QC + 2) * WLD];
  __shared__ double rot_cs[QC];
  __shared__ cplx rot_sn[QC];
  const int prob = blockIdx.x;
  const int k = kdim[prob];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  EigWs w = carve(ws, wstride, prob, kmax);
  const cplx* Ai = At + (long long)prob * sin_;
  const cplx* Bi = Bt + (long long)prob * sin_;
  cplx *H = w.A, *LU = w.L, *Z = w.V, *X = w.T;
  int* piv = reinterpret_cast<int*>(w.d);
  const int ld = kmax;
  for (int e = tid; e < k * k; e += GT) {
    int r = e / k, c = e % k;
    LU[r * ld + c] = Bi[(long long)r * ldin + c];
    H[r * ld + c] = Ai[(long long)r * ldin + c];
    Z[r * ld + c] = cmk(r == c ? 1.0 : 0.0, 0.0);
  }
  if (tid == 0) s_int[3] = 0;
  __syncthreads();
  EIG_MARK(0);
  // 1. LU of B~ with partial pivoting; apply the same row swaps to H
  for (int j = 0; j < k; ++j) {
    double best = -1.0; int bi = j;
    for (int r = j + tid; r < k; r += GT) {
      double v = cabs1(LU[r * ld + j]);
      if (v > best) { best = v; bi = r; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { rv[wid] = best; ri[wid] = bi; }
    __syncthreads();
    if (wid == 0) {
      best = lane < GT / 32 ? rv[lane] : -1.0;
      bi = lane < GT / 32 ? ri[lane] : k;
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) { s_int[0] = bi; piv[j] = bi; if (best == 0.0) s_int[3] = j + 1; }
    }
    __syncthreads();
    const int p = s_int[0];
    if (p != j) {
      for (int c = tid; c < k; c += GT) {
        cplx t = LU[j * ld + c]; LU[j * ld + c] = LU[p * ld + c]; LU[p * ld + c] = t;
        t = H[j * ld + c]; H[j * ld + c] = H[p * ld + c]; H[p * ld + c] = t;
      }
    }
    __syncthreads();
    const cplx pv = LU[j * ld + j];
    if (pv.x != 0.0 || pv.y != 0.0) {
      const cplx rp = crecip(pv);
      for (int r = j + 1 + tid; r < k; r += GT) LU[r * ld + j] = cmul(LU[r * ld + j], rp);
      __syncthreads();
      const int m = k - j - 1;
      batched_rmw<4>(m * m, GT,
          [&](int e) -> cplx* { return LU + (j + 1 + e / m) * ld + j + 1 + e % m; },
          [&](int e, cplx v) { cfms(v, LU[(j + 1 + e / m) * ld + j], LU[j * ld + j + 1 + e % m]); return v; });
    }
    __syncthreads();
  }
  if (s_int[3]) {
    if (tid == 0) info[prob] = s_int[3];
    return;
  }
  EIG_MARK(1);
  // solve L U M = P A (column per thread), M into H
  for (int c = tid; c < k; c += GT) {
    for (int i = 0; i < k; ++i) {
      cplx v = H[i * ld + c];
      for (int l = 0; l < i; ++l) cfms(v, LU[i * ld + l], H[l * ld + c]);
      H[i * ld + c] = v;
    }
    for (int i = k - 1; i >= 0; --i) {
      cplx v = H[i * ld + c];
      for (int l = i + 1; l < k; ++l) cfms(v, LU[i * ld + l], H[l * ld + c]);
      H[i * ld + c] = cdiv(v, LU[i * ld + i]);
    }
  }
  __syncthreads();
  EIG_MARK(2);
  // 2. Householder Hessenberg reduction H <- Q^H H Q, Z <- Z Q.  The two
  // matrix-vector products per column are split into 16-deep slices (many
  // independent L2 loads in flight per thread) with fixed-order partial sums.
  cplx* v = w.vec;          // Householder vector (length k)
  cplx* wv = w.vec + kmax;  // work vectors (length 2k)
  cplx* part = w.T;         // partial sums (<= 2k x ceil(k/16)), T is free until step 4
  for (int j = 0; j + 2 < k; ++j) {
    const int m = k - j - 1;  // rows j+1 .. k-1
    double xs = 0.0;
    for (int r = j + 2 + tid; r < k; r += GT) xs += cabs2(H[r * ld + j]);
    xs = block_sum(xs, red);
    const cplx alpha = H[(j + 1) * ld + j];
    if (xs != 0.0 || alpha.y != 0.0) {
      const double xnorm = sqrt(xs);
      double beta = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xnorm * xnorm);
      beta = alpha.x >= 0.0 ? -beta : beta;
      const cplx tau = cmk((beta - alpha.x) / beta, -alpha.y / beta);
      const cplx scal = crecip(cmk(alpha.x - beta, alpha.y));
      for (int r = tid; r < m; r += GT) v[r] = r == 0 ? cmk(1.0, 0.0) : cmul(H[(j + 1 + r) * ld + j], scal);
      __syncthreads();
      if (tid == 0) H[(j + 1) * ld + j] = cmk(beta, 0.0);
      for (int r = j + 2 + tid; r < k; r += GT) H[r * ld + j] = cmk(0.0, 0.0);
      // left: wv[c] = sum_r conj(v_r) H[j+1+r][c], c in j+1..k-1 (slices of 16 rows)
      const int nc = k - j - 1, ns = (m + 15) / 16;
      for (int e = tid; e < nc * ns; e += GT) {
        const int c = j + 1 + e % nc, sl = e / nc;
        const int r0 = sl * 16, r1 = min(m, r0 + 16);
        cplx acc = cmk(0.0, 0.0);
#pragma unroll 8
        for (int r = r0; r < r1; ++r) cfma(acc, cconj(v[r]), H[(j + 1 + r) * ld + c]);
        part[sl * (2 * kmax) + c] = acc;
      }
      __syncthreads();
      for (int c = j + 1 + tid; c < k; c += GT) {
        cplx acc = cmk(0.0, 0.0);
        for (int sl = 0; sl < ns; ++sl) acc = cadd(acc, part[sl * (2 * kmax) + c]);
        wv[c] = acc;
      }
      __syncthreads();
      const cplx ct = cconj(tau);
      batched_rmw<4>(m * nc, GT,
          [&](int e) -> cplx* { return H + (j + 1 + e / nc) * ld + j + 1 + e % nc; },
          [&](int e, cplx x) { cfms(x, cmul(ct, v[e / nc]), wv[j + 1 + e % nc]); return x; });
      __syncthreads();
      // right: wv[r] = sum_i M[r][j+1+i] v_i over the rows of H and Z (slices of 16 columns)
      for (int e = tid; e < 2 * k * ns; e += GT) {
        const int rowi = e % (2 * k), sl = e / (2 * k);
        const cplx* M = rowi < k ? H : Z;
        const int rr = rowi < k ? rowi : rowi - k;
        const int i0 = sl * 16, i1 = min(m, i0 + 16);
        cplx acc = cmk(0.0, 0.0);
#pragma unroll 8
        for (int i = i0; i < i1; ++i) cfma(acc, M[rr * ld + j + 1 + i], v[i]);
        part[sl * (2 * kmax) + rowi] = acc;
      }
      __syncthreads();
      for (int rowi = tid; rowi < 2 * k; rowi += GT) {
        cplx acc = cmk(0.0, 0.0);
        for (int sl = 0; sl < ns; ++sl) acc = cadd(acc, part[sl * (2 * kmax) + rowi]);
        wv[rowi] = acc;
      }
      __syncthreads();
      batched_rmw<4>(2 * k * m, GT,
          [&](int e) -> cplx* { const int rowi = e / m; return (rowi < k ? H + rowi * ld : Z + (rowi - k) * ld) + j + 1 + e % m; },
          [&](int e, cplx x) { cfms(x, cmul(tau, wv[e / m]), cconj(v[e % m])); return x; });
      __syncthreads();
    }
  }
  EIG_MARK(3);
  // 3. single-shift QR on the Hessenberg matrix (full Schur form + Z)
  int ihi = k - 1;
  const int itmax = 30 * (k > 10 ? k : 10);
  int fail = 0;
  long long n_sweeps = 0, n_rot = 0, t_win = 0, t_chain = 0, t_def = 0;
  while (ihi >= 0) {
    int l = 0;
    int its = 0;
    for (; its <= itmax; ++its) {
      // find the largest kk in (l, ihi] with a negligible subdiagonal
      int found = l;
      for (int kk = l + 1 + tid; kk <= ihi; kk += GT) {
        const double hs = cabs1(H[kk * ld + kk - 1]);
        double tst = cabs1(H[(kk - 1) * ld + kk - 1]) + cabs1(H[kk * ld + kk]);
        if (tst == 0.0) {
          if (kk - 2 >= l) tst += fabs(H[(kk - 1) * ld + kk - 2].x);
          if (kk + 1 <= ihi) tst += fabs(H[(kk + 1) * ld + kk].x);
        }
        bool neg = hs <= 1e-300;
        if (!neg && hs <= EPS * tst) {
          // zlahqr's Ahues & Tisseur test: also deflate when the off-diagonal
          // product is negligible against the local eigenvalue gap
          const double h01 = cabs1(H[(kk - 1) * ld + kk]);
          const double ab = fmax(hs, h01), ba = fmin(hs, h01);
          const double hkk = cabs1(H[kk * ld + kk]);
          const double dd = cabs1(csub(H[(kk - 1) * ld + kk - 1], H[kk * ld + kk]));
          const double aa = fmax(hkk, dd), bb = fmin(hkk, dd);
          const double s = aa + ab;
          neg = ba * (ab / s) <= fmax(1e-300, EPS * (bb * (aa / s)));
        }
        if (neg) found = max(found, kk);
      }
      for (int o = 16; o > 0; o >>= 1) found = max(found, __shfl_xor_sync(0xffffffffu, found, o));
      if (lane == 0) ri[wid] = found;
      __syncthreads();
      if (tid == 0) {
        int f = l;
        for (int q = 0; q < GT / 32; ++q) f = max(f, ri[q]);
        s_int[1] = f;
        if (f > l) H[f * ld + f - 1] = cmk(0.0, 0.0);
      }
      __syncthreads();
      l = s_int[1];
      if (l >= ihi) break;
      // shift
      if (tid == 0) {
        cplx mu;
        if (its == 10) {
          mu = cadd(cmk(0.75 * fabs(H[(l + 1) * ld + l].x), 0.0), H[l * ld + l]);
        } else if (its == 20) {
          mu = cadd(cmk(0.75 * fabs(H[ihi * ld + ihi - 1].x), 0.0), H[ihi * ld + ihi]);
        } else {
          cplx t = H[ihi * ld + ihi];
          cplx u = cmul(csqrt_(H[(ihi - 1) * ld + ihi]), csqrt_(H[ihi * ld + ihi - 1]));
          double s = cabs1(u);
          if (s != 0.0) {
            cplx x = cscale(csub(H[(ihi - 1) * ld + ihi - 1], t), 0.5);
            double sx = cabs1(x);
            s = fmax(s, sx);
            cplx xs_ = cscale(x, 1.0 / s), us = cscale(u, 1.0 / s);
            cplx y = cscale(csqrt_(cadd(cmul(xs_, xs_), cmul(us, us))), s);
            if (sx > 0.0) {
              cplx xn = cscale(x, 1.0 / sx);
              if (xn.x * y.x + xn.y * y.y < 0.0) y = cmk(-y.x, -y.y);
            }
            t = csub(t, cmul(u, cdiv(u, cadd(x, y))));
          }
          mu = t;
        }
        s_c[0] = mu;
      }
      __syncthreads();
      const cplx mu = s_c[0];
      ++n_sweeps;
      n_rot += ihi - l;
      // QR sweep over rows/cols l..ihi in chunks of QC rotations: warp 0 chases
      // the bulge through a shared-memory window (every entry the chain reads
      // lives there); afterwards all warps apply the chunk's rotations to the
      // far parts of H (left: window rows right of the window; right: rows
      // above it) and to Z, one carry per row/column, no further syncs.
      for (int m0 = l; m0 < ihi; m0 += QC) {
        long long tq0 = clock64();
        const int m1 = min(m0 + QC, ihi);
        const int wr0 = m0, wr1 = min(m1 + 1, ihi);
        const int wc0 = (m0 > l) ? m0 - 1 : l, wc1 = min(m1 + 1, ihi);
        const int nwr = wr1 - wr0 + 1, nwc = wc1 - wc0 + 1;
        for (int e = tid; e < nwr * nwc; e += GT) {
          const int r = e / nwc, cc = e % nwc;
          win[r * WLD + cc] = H[(wr0 + r) * ld + wc0 + cc];
        }
        __syncthreads();
        long long tq1 = clock64();
        if (wid == 0) {
#define W_(r, c) win[((r) - wr0) * WLD + (c) - wc0]
          for (int m = m0; m < m1; ++m) {
            // every lane forms the rotation itself (no broadcast); lane 0 records it
            cplx x, y;
            if (m == l) { x = csub(W_(l, l), mu); y = W_(l + 1, l); }
            else { x = W_(m, m - 1); y = W_(m + 1, m - 1); }
            const double nx2 = cabs2(x), ny2 = cabs2(y);
            double c; cplx sn, r;
            if (ny2 == 0.0) { c = 1.0; sn = cmk(0.0, 0.0); r = x; }
            else if (nx2 == 0.0) { const double ay = sqrt(ny2); c = 0.0; sn = cscale(cconj(y), 1.0 / ay); r = cmk(ay, 0.0); }
            else {
              const double ax = sqrt(nx2);
              const double inv = rsqrt(nx2 + ny2);
              c = ax * inv;
              const cplx ph = cscale(x, 1.0 / ax);
              sn = cscale(cmul(ph, cconj(y)), inv);
              r = cscale(ph, (nx2 + ny2) * inv);
            }
            __syncwarp();
            if (lane == 0) {
              if (m > l) { W_(m, m - 1) = r; W_(m + 1, m - 1) = cmk(0.0, 0.0); }
              rot_cs[m - m0] = c;
              rot_sn[m - m0] = sn;
            }
            const cplx snc = cconj(sn);
            for (int col = m + lane; col <= wc1; col += 32) {
              const cplx a = W_(m, col), b = W_(m + 1, col);
              W_(m, col) = cadd(cscale(a, c), cmul(sn, b));
              W_(m + 1, col) = csub(cscale(b, c), cmul(snc, a));
            }
            __syncwarp();
            const int rmax = min(m + 2, wr1);
            for (int r = wr0 + lane; r <= rmax; r += 32) {
              const cplx a = W_(r, m), b = W_(r, m + 1);
              W_(r, m) = cadd(cscale(a, c), cmul(snc, b));
              W_(r, m + 1) = csub(cscale(b, c), cmul(sn, a));
            }
            __syncwarp();
          }
#undef W_
        }
        __syncthreads();
        long long tq2 = clock64();
        for (int e = tid; e < nwr * nwc; e += GT) {
          const int r = e / nwc, cc = e % nwc;
          H[(wr0 + r) * ld + wc0 + cc] = win[r * WLD + cc];
        }
        const int na = k - 1 - wc1, nb = wr0, nz = k;
        const int nrot = m1 - m0;
        for (int w = tid; w < na + nb + nz; w += GT) {
          cplx* M;
          long long base, step;
          bool left;
          if (w < na) { M = H; base = (long long)m0 * ld + wc1 + 1 + w; step = ld; left = true; }
          else {
            const int r = (w < na + nb) ? w - na : w - na - nb;
            M = (w < na + nb) ? H : Z;
            base = (long long)r * ld + m0; step = 1; left = false;
          }
          cplx xs[QC + 1];
#pragma unroll
          for (int q = 0; q <= QC; ++q)
            if (q <= nrot) xs[q] = M[base + q * step];
#pragma unroll
          for (int q = 0; q < QC; ++q) {
            if (q < nrot) {
              const double c = rot_cs[q];
              const cplx sn = left ? rot_sn[q] : cconj(rot_sn[q]);
              const cplx x = xs[q], y = xs[q + 1];
              xs[q] = cadd(cscale(x, c), cmul(sn, y));
              xs[q + 1] = csub(cscale(y, c), cmul(cconj(sn), x));
            }
          }
#pragma unroll
          for (int q = 0; q <= QC; ++q)
            if (q <= nrot) M[base + q * step] = xs[q];
        }
        __syncthreads();
        long long tq3 = clock64();
        t_win += tq1 - tq0; t_chain += tq2 - tq1; t_def += tq3 - tq2;
        __syncthreads();
      }
    }
    if (its > itmax) { fail = ihi + 1; break; }
    ihi = l - 1;
  }
  if (blockIdx.x == 0 && tid == 0) {
    g_eig_phase[8] = n_sweeps; g_eig_phase[9] = n_rot;
    g_eig_phase[10] = t_win; g_eig_phase[11] = t_chain; g_eig_phase[12] = t_def;
  }
  if (fail) {
    if (tid == 0) info[prob] = -fail;
    return;
  }
  // zero below the diagonal (Schur form is upper triangular)
  for (int e = tid; e < k * k; e += GT) {
    int r = e / k, c = e % k;
    if (r > c) H[r * ld + c] = cmk(0.0, 0.0);
  }
  __syncthreads();
  EIG_MARK(4);
  // 4. eigenvectors of T by back substitution: X[:, e]
  double tnorm = 0.0;
  for (int e = tid; e < k * k; e += GT) tnorm = fmax(tnorm, cabs1(H[e / k * ld + e % k]));
  tnorm = block_max(tnorm, red);
  const double smlnum = 1e-300 * (double)k / EPS;
  for (int e = tid; e < k; e += GT) {
    const cplx te = H[e * ld + e];
    const double smin = fmax(EPS * cabs1(te), smlnum);
    for (int r = k - 1; r > e; --r) X[r * ld + e] = cmk(0.0, 0.0);
    X[e * ld + e] = cmk(1.0, 0.0);
    for (int r = e - 1; r >= 0; --r) {
      cplx acc = H[r * ld + e];
      for (int c = r + 1; c < e; ++c) cfma(acc, H[r * ld + c], X[c * ld + e]);
      cplx den = csub(H[r * ld + r], te);
      if (cabs1(den) < smin) den = cmk(smin, 0.0);
      X[r * ld + e] = cdiv(cmk(-acc.x, -acc.y), den);
    }
  }
  __syncthreads();
  EIG_MARK(5);
  // eigenvalue order: ascending by (re, im)
  for (int i = tid; i < k; i += GT) {
    const cplx li = H[i * ld + i];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const cplx lj = H[j * ld + j];
      rank += (lj.x < li.x) || (lj.x == li.x && (lj.y < li.y || (lj.y == li.y && j < i)));
    }
    piv[i] = rank;
    lam[(long long)prob * kmax + rank] = li;
  }
  __syncthreads();
  // vectors Z X, unit 2-norm; column e of the Schur vectors -> S[:, rank]
  cplx* Sp = S + (long long)prob * sS;
  for (int e = wid; e < k; e += GT / 32) {
    double nrm = 0.0;
    for (int r = lane; r < k; r += 32) {
      cplx acc = cmk(0.0, 0.0);
      for (int c = 0; c <= e; ++c) cfma(acc, Z[r * ld + c], X[c * ld + e]);
      Sp[(long long)r * lds + piv[e]] = acc;
      nrm += cabs2(acc);
    }
    nrm = sqrt(warp_sum(nrm));
    const double inv = nrm > 0.0 ? 1.0 / nrm : 1.0;
    __syncwarp();
    for (int r = lane; r < k; r += 32) {
      cplx* p = Sp + (long long)r * lds + piv[e];
      *p = cscale(*p, inv);
    }
  }
  EIG_MARK(6);
  if (tid == 0) info[prob] = 0;
}

}  // namespace

// Workspace bytes per problem for cirr_small_eig.
static long long small_eig_slot(int kmax) {
  return ((long long)kmax * kmax * 16 * 4 + (long long)kmax * 16 * 4 + (long long)kmax * 8 * 4 + 256 + 255) / 256 * 256;
}
// per-problem share of the cooperative-SVD path's shared region (Qt, sigma,
// order, kept, sweeps and cirr_orth's own workspace), placed after the slots
static long long small_eig_extra(int kmax) {
  return ((long long)kmax * kmax * 16 * 3 + (long long)kmax * 16 * 2 + 8192 + 255) / 256 * 256;
}
CIRR_API long long cirr_small_eig_ws_bytes(int kmax) { return small_eig_slot(kmax) + small_eig_extra(kmax); }

// Eigen-decomposition of nprob projected pencils (A~, B~), each k_b x k_b
// (kdim device array, k_b <= kmax <= 1024), row-major with ld ldin and batch
// stride sin_.  hermitian != 0: Hermitian-definite path (eigh); else general
// (eig).  lam: nprob x kmax complex (sorted); S: eigenvectors as columns;
// info: 0 ok, >0 Cholesky/LU failure at that 1-based index, <0 QR failure.
CIRR_API int cirr_small_eig(int hermitian, const cplx* At, const cplx* Bt, long long ldin, long long sin_,
                            const int* kdim, int kmax, int nprob, void* ws, cplx* lam, cplx* S, long long lds,
                            long long sS, int* info, cudaStream_t stream) {
  if (kmax <= 0 || kmax > 1024 || nprob <= 0) return CIRR_EINVAL;
  // per-problem slots of small_eig_slot bytes, then the shared region (the
  // caller allocates nprob x cirr_small_eig_ws_bytes)
  const long long wstride = small_eig_slot(kmax);
  static const bool coop = !(getenv("CIRR_HERM_COOP") && getenv("CIRR_HERM_COOP")[0] == '0');
  if (hermitian && kmax > 78 && nprob <= 64 && coop) {
    // one-sided Jacobi of the HPD A' = L^-1 A~ L^-H across the whole GPU
    // (cirr_orth's cooperative kernel) instead of one CTA per problem;
    // MODE 2 checks every pair and MODE 3 redoes a problem whose A' was not
    // definite
    unsigned char* shared = reinterpret_cast<unsigned char*>(ws) + (long long)nprob * wstride;
    const long long kk = (long long)kmax * kmax;
    cplx* Qt = reinterpret_cast<cplx*>(shared);
    double* sigma = reinterpret_cast<double*>(Qt + (long long)nprob * kk);
    int* order = reinterpret_cast<int*>(sigma + (long long)nprob * kmax);
    int* kept = order + (long long)nprob * kmax;
    int* sweeps = kept + nprob;
    unsigned char* ows = reinterpret_cast<unsigned char*>(((uintptr_t)(sweeps + 1) + 255) & ~(uintptr_t)255);
    if ((ows - shared) + cirr_orth_ws_bytes(kmax, nprob) > (long long)nprob * small_eig_extra(kmax)) return CIRR_EINVAL;
    herm_eig_kernel<false, 1><<<nprob, ET, 0, stream>>>(At, Bt, ldin, sin_, kdim, kmax, ws, wstride, lam, S, lds,
                                                        sS, info);
    CIRR_CHECK_LAUNCH();
    // W = the T block of each slot (kmax x kmax rows, slot stride)
    cplx* W0 = reinterpret_cast<cplx*>(reinterpret_cast<unsigned char*>(ws) + 3 * kk * 16);
    CIRR_TRY(cirr_orth(W0, kmax, wstride / 16, kmax, kmax, nprob, 0.0, sigma, order, kept, Qt, kmax, kk, ows, sweeps,
                       stream));
    herm_eig_kernel<false, 2><<<nprob, ET, 0, stream>>>(At, Bt, ldin, sin_, kdim, kmax, ws, wstride, lam, S, lds,
                                                        sS, info, Qt, sigma);
    CIRR_CHECK_LAUNCH();
    herm_eig_kernel<false, 3><<<nprob, ET, 0, stream>>>(At, Bt, ldin, sin_, kdim, kmax, ws, wstride, lam, S, lds,
                                                        sS, info);
    CIRR_CHECK_LAUNCH();
    return 0;
  }
  if (hermitian) {
    // A and V in shared memory for kmax <= 78 (2 kmax (kmax+1) complex <= 193 KB next
    // to the 16 KB of static rotation tables); CIRR_HERM_SMEM=0 disables
    static const bool hs = !(getenv("CIRR_HERM_SMEM") && getenv("CIRR_HERM_SMEM")[0] == '0');
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(herm_eig_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 78 * 79 * 16);
      attr = true;
    }
    if (hs && kmax <= 78)
      herm_eig_kernel<true><<<nprob, ET, (size_t)2 * kmax * (kmax + 1) * sizeof(cplx), stream>>>(
          At, Bt, ldin, sin_, kdim, kmax, ws, wstride, lam, S, lds, sS, info);
    else
      herm_eig_kernel<false><<<nprob, ET, 0, stream>>>(At, Bt, ldin, sin_, kdim, kmax, ws, wstride, lam, S, lds, sS,
                                                      info);
  } else
    gen_eig_kernel<<<nprob, GT, 0, stream>>>(At, Bt, ldin, sin_, kdim, kmax, ws, wstride, lam, S, lds, sS, info);
  CIRR_CHECK_LAUNCH();
  return 0;
}

// debug: clock64 phase stamps of the last gen_eig launch (problem 0)
CIRR_API int cirr_small_eig_phases(long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_eig_phase, sizeof(long long) * 16);
}
