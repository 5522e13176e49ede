// K6 for refinement rounds (non-Hermitian): the projected eigenproblem solved
// by Newton refinement of a known approximate eigenbasis instead of the
// sequential Hessenberg QR.
//
// In a CIRR refinement round (solvers.py:200-205 -> 178-198) the block is
// S = P X, the filtered Ritz vectors of the previous round, so its columns are
// already close to eigenvectors of the new projected pencil and, in the basis
// Q of range(S), W0 = Q^H S is an approximate eigenvector matrix of
// M = B~^-1 A~.  With T = W^-1 M W = D + E (D = diag(T)) the first-order
// correction W <- W (I + F), F_ij = T_ij / (T_jj - T_ii), squares the
// off-diagonal part per step (Newton on the eigendecomposition, the classical
// perturbation update).  Every step is batched DMMA work over the whole GPU:
// M W and W (I + F) on cirr_gemm, W^-1 (M W) on the batched LU and solve,
// plus one small kernel per problem for F and the convergence test -- no
// one-CTA sequential sweep.  Once max_{i != j} |T_ij| reaches the rounding
// floor the eigenvalues are T_jj + sum_i T_ji T_ij / (T_jj - T_ii) and the
// eigenvectors the unit-normalised columns of W.
//
// The few columns of W0 that are not near eigenvectors (Ritz pairs of the
// previous round that had not converged: 1-5 of ~120 per contour on config 4,
// the rest have max_i |T_ij| <= 1e-5 ||T||) are first replaced by the
// eigenvectors of their own block: with b those columns, T_bg ~ 0 (the good
// columns are near-invariant), so eig(T) ~ eig(T_gg) u eig(T_bb); the k_b x k_b
// eigenproblem (k_b <= 32) goes through the QR path and W_b <- W_b V_bb.  The
// Newton steps then converge for every column, the first one adding to each
// rotated column its component along the good ones, (mu - D_g)^-1 T_gb.
//
// A problem whose basis does not converge (a near-degenerate pair, or a W0
// too far from an eigenbasis) reports info = -1 and the caller solves it with
// cirr_gen_eig_values / cirr_gen_eig_vectors (QR), so the result never depends
// on the refinement converging.  Output conventions are those of the QR path:
// eigenvalues sorted by (re, im) like numpy's sort, unit 2-norm eigenvectors
// in the same order.
#include "common.cuh"
#include <utility>

namespace {

constexpr int RT = 256;  // threads per problem; k <= 256
constexpr int KB = 32;   // most columns replaced from the small block eigenproblem
constexpr double TAU_BAD = 1e-3;   // max_i |T_ij| > TAU_BAD * ||T||: column j is not near an eigenvector

// debug: per problem (first 8) the step at which it converged (-1: not), and
// the number of columns the block step replaced
__device__ int g_refine_stats[16];

__device__ __forceinline__ long long moff(int p, int kmax) { return (long long)p * kmax * kmax; }

// W[p] = (W0h[p])^H with unit-norm columns; identity on the padding.
__global__ void __launch_bounds__(RT) refine_init_kernel(const cplx* __restrict__ W0h, long long ldw,
                                                         long long sw, const int* __restrict__ kdim, int kmax,
                                                         cplx* __restrict__ W, int* __restrict__ state,
                                                         double* __restrict__ offprev) {
  const int p = blockIdx.x, j = threadIdx.x;
  const int k = kdim[p];
  cplx* Wp = W + moff(p, kmax);
  if (j == 0) {
    state[p] = 0;
    offprev[p] = 1e300;
  }
  if (j >= kmax) return;
  if (j < k) {
    const cplx* row = W0h + (long long)p * sw + (long long)j * ldw;   // column j of W0
    double nrm = 0.0;
    for (int i = 0; i < k; ++i) nrm += cabs2(row[i]);
    nrm = sqrt(nrm);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int i = 0; i < kmax; ++i) Wp[(long long)i * kmax + j] = i < k ? cscale(cconj(row[i]), inv) : cmk(0.0, 0.0);
  } else {
    for (int i = 0; i < kmax; ++i) Wp[(long long)i * kmax + j] = cmk(i == j ? 1.0 : 0.0, 0.0);
  }
}

// B~ padded with the identity (cirr_zgetrf_batched then factors a regular matrix)
__global__ void refine_pad_kernel(cplx* B, const int* kdim, int kmax) {
  const int p = blockIdx.x;
  for (int i = kdim[p] + threadIdx.x; i < kmax; i += blockDim.x) B[moff(p, kmax) + (long long)i * kmax + i] = cmk(1.0, 0.0);
}

__global__ void refine_iota_kernel(int* v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

// Columns of T = W0^-1 M W0 that are far from e_j: their list, the block
// T_bb (KB x KB, zero padded, k_b >= 1 so the QR path always has a problem:
// k_b = 0 gets a 1 x 1 dummy), the identity B operand and the selection of
// all k_b eigenvectors.  k_b > KB: state = 2 (fall back).
__global__ void __launch_bounds__(RT) refine_classify_kernel(const cplx* __restrict__ T, const int* __restrict__ kdim,
                                                             int kmax, int* __restrict__ state, int* __restrict__ nbad,
                                                             int* __restrict__ bad, cplx* __restrict__ Tbb,
                                                             cplx* __restrict__ Ibb, int* __restrict__ kdim_b,
                                                             int* __restrict__ sel_b) {
  __shared__ double red[32];
  __shared__ int cnt;
  __shared__ int list[RT];
  const int p = blockIdx.x, j = threadIdx.x;
  const int k = kdim[p];
  const cplx* Tp = T + moff(p, kmax);
  double c = 0.0, dm = 0.0;
  if (j < k) {
    dm = cabs(Tp[(long long)j * kmax + j]);
    for (int i = 0; i < k; ++i)
      if (i != j) c = fmax(c, cabs(Tp[(long long)i * kmax + j]));
  }
  const double scale = fmax(block_max(dm, red), block_max(c, red));
  if (j == 0) cnt = 0;
  __syncthreads();
  // ordered list of the bad columns (ballot per warp, prefix over warps)
  const bool isbad = j < k && !(c <= TAU_BAD * scale);
  for (int w = 0; w < RT / 32; ++w) {
    if ((j >> 5) == w) {
      const unsigned m = __ballot_sync(0xffffffffu, isbad);
      if (isbad) list[cnt + __popc(m & ((1u << (j & 31)) - 1u))] = j;
      __syncwarp();
      if ((j & 31) == 0) cnt += __popc(m);
    }
    __syncthreads();
  }
  const int kb = cnt;
  cplx* Tb = Tbb + (long long)p * KB * KB;
  cplx* Ib = Ibb + (long long)p * KB * KB;
  for (int e = j; e < KB * KB; e += RT) {
    const int r = e / KB, q = e % KB;
    cplx v = cmk(0.0, 0.0);
    if (kb == 0 || kb > KB) v = cmk(r == 0 && q == 0 ? 1.0 : 0.0, 0.0);
    else if (kb <= KB && r < kb && q < kb) v = Tp[(long long)list[r] * kmax + list[q]];
    Tb[e] = v;
    Ib[e] = cmk(r == q ? 1.0 : 0.0, 0.0);
  }
  if (j < KB) sel_b[(long long)p * KB + j] = j;
  if (j < kb && j < KB) bad[(long long)p * KB + j] = list[j];
  if (j == 0 && p < 8) {
    g_refine_stats[p] = -1;
    g_refine_stats[8 + p] = kb;
  }
  if (j == 0) {
    // more than KB such columns: no block step, the Newton steps alone decide
    nbad[p] = kb <= KB ? kb : 0;
    kdim_b[p] = (kb == 0 || kb > KB) ? 1 : kb;
    if (!(scale > 0.0)) state[p] = 2;
  }
}

// The bad columns replaced by the eigenvectors of their block, W_b <- W_b V,
// and the matching rows of the inverse, Yh_b <- V^-1 Yh_b (V^-1 by
// Gauss-Jordan with partial pivoting in shared memory, k_b <= KB).  Thread t
// rewrites row t of W and column t of Yh, so no thread reads what another
// writes.
__global__ void __launch_bounds__(RT) refine_rotate_kernel(cplx* __restrict__ W, cplx* __restrict__ Yh,
                                                           const int* __restrict__ kdim, int kmax,
                                                           const int* __restrict__ nbad, const int* __restrict__ bad,
                                                           const cplx* __restrict__ Vbb, const int* __restrict__ info_b,
                                                           int* __restrict__ state) {
  __shared__ cplx Aw[KB * KB], Vi[KB * KB];
  __shared__ int cols[KB];
  __shared__ int piv;
  __shared__ int fail;
  const int p = blockIdx.x, t = threadIdx.x;
  const int kb = nbad[p];
  if (kb == 0 || kb > KB || state[p] != 0) return;
  if (info_b[p] != 0) {
    if (t == 0) state[p] = 2;
    return;
  }
  const cplx* V = Vbb + (long long)p * KB * KB;   // ld KB
  for (int e = t; e < KB * KB; e += RT) {
    const int r = e / KB, q = e % KB;
    Aw[e] = (r < kb && q < kb) ? V[e] : cmk(0.0, 0.0);   // Gauss-Jordan works on a copy
    Vi[e] = cmk(r == q ? 1.0 : 0.0, 0.0);
  }
  if (t < kb) cols[t] = bad[(long long)p * KB + t];
  if (t == 0) fail = 0;
  __syncthreads();
  for (int c = 0; c < kb; ++c) {
    if (t < 32) {
      double best = -1.0;
      int bi = c;
      for (int r = c + t; r < kb; r += 32) {
        const double a = cabs1(Aw[r * KB + c]);
        if (a > best) { best = a; bi = r; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (t == 0) {
        piv = bi;
        if (!(best > 0.0)) fail = 1;
      }
    }
    __syncthreads();
    if (fail) break;
    const int pr = piv;
    if (pr != c && t < 2 * KB) {
      cplx* M = t < KB ? Aw : Vi;
      const int q = t % KB;
      const cplx tmp = M[c * KB + q];
      M[c * KB + q] = M[pr * KB + q];
      M[pr * KB + q] = tmp;
    }
    __syncthreads();
    const cplx inv = crecip(Aw[c * KB + c]);
    __syncthreads();
    if (t < 2 * KB) {
      cplx* M = t < KB ? Aw : Vi;
      const int q = t % KB;
      M[c * KB + q] = cmul(M[c * KB + q], inv);
    }
    __syncthreads();
    for (int e = t; e < 2 * KB * KB; e += RT) {
      const int r = (e % (KB * KB)) / KB, q = e % KB;
      if (r == c || r >= kb) continue;
      cplx* M = e < KB * KB ? Aw : Vi;
      const cplx f = Aw[r * KB + c];
      // Aw column c itself is read by every row: eliminate it last (below)
      if (e < KB * KB && q == c) continue;
      cfms(M[r * KB + q], f, M[c * KB + q]);
    }
    __syncthreads();
    if (t < kb && t != c) Aw[t * KB + c] = cmk(0.0, 0.0);
    __syncthreads();
  }
  if (fail) {
    if (t == 0) state[p] = 2;
    return;
  }
  const int k = kdim[p];
  if (t >= k) return;
  cplx old[KB];
  {  // row t of W: W[t, cols] <- W[t, cols] V
    cplx* row = W + moff(p, kmax) + (long long)t * kmax;
#pragma unroll
    for (int m = 0; m < KB; ++m) old[m] = m < kb ? row[cols[m]] : cmk(0.0, 0.0);
    for (int l = 0; l < kb; ++l) {
      cplx acc = cmk(0.0, 0.0);
#pragma unroll
      for (int m = 0; m < KB; ++m)
        if (m < kb) cfma(acc, old[m], V[m * KB + l]);
      row[cols[l]] = acc;
    }
  }
  {  // column t of Yh: Yh[cols, t] <- V^-1 Yh[cols, t]
    cplx* Yp = Yh + moff(p, kmax);
#pragma unroll
    for (int m = 0; m < KB; ++m) old[m] = m < kb ? Yp[(long long)cols[m] * kmax + t] : cmk(0.0, 0.0);
    for (int l = 0; l < kb; ++l) {
      cplx acc = cmk(0.0, 0.0);
#pragma unroll
      for (int m = 0; m < KB; ++m)
        if (m < kb) cfma(acc, Vi[l * KB + m], old[m]);
      Yp[(long long)cols[l] * kmax + t] = acc;
    }
  }
}

// X = a I on the k x k block, I on the padding
__global__ void refine_fill_identity_kernel(cplx* X, const int* kdim, int kmax, double a) {
  const int p = blockIdx.y;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)kmax * kmax) return;
  const int r = (int)(e / kmax), q = (int)(e % kmax);
  X[moff(p, kmax) + e] = cmk(r == q ? (r < kdim[p] ? a : 1.0) : 0.0, 0.0);
}

// One problem per CTA, thread j owns column j of T = W^-1 M W:
//   F = (T_ij / (T_jj - T_ii))_{i != j} as I + F and I - F, the convergence test, and on
//   convergence the eigenvalues with their second-order correction.
// state: 0 iterating, 1 converged, 2 failed.  Converged / failed problems get
// F = 0, so later steps leave W unchanged (exactly: 1 * w + 0 * ... in DMMA).
__global__ void __launch_bounds__(RT) refine_update_kernel(const cplx* __restrict__ T, const int* __restrict__ kdim,
                                                           int kmax, const int* __restrict__ wluinfo,
                                                           int* __restrict__ state, double* __restrict__ offprev,
                                                           cplx* __restrict__ F, cplx* __restrict__ Fm,
                                                           cplx* __restrict__ lamd, int it, int last) {
  __shared__ cplx d[RT];
  __shared__ double red[32];
  __shared__ int st_s;
  const int p = blockIdx.x, j = threadIdx.x;
  const int k = kdim[p];
  const cplx* Tp = T + moff(p, kmax);
  cplx* Fp = F + moff(p, kmax);
  cplx* Fmp = Fm + moff(p, kmax);
  if (j < kmax) d[j] = Tp[(long long)j * kmax + j];
  if (j == 0) st_s = state[p];
  __syncthreads();
  int st = st_s;
  if (st == 0 && wluinfo[p] != 0) st = 2;   // W singular: not an eigenbasis
  double off = 0.0, eta = 0.0, dmax = 0.0;
  cplx corr = cmk(0.0, 0.0);
  if (st == 0 && j < k) {
    const cplx dj = d[j];
    dmax = cabs(dj);
    for (int i = 0; i < k; ++i) {
      if (i == j) continue;
      const cplx tij = Tp[(long long)i * kmax + j];
      const cplx gap = csub(dj, d[i]);
      const double a = cabs(tij), g = cabs(gap);
      off = fmax(off, a);
      eta = fmax(eta, g > 0.0 ? a / g : (a > 0.0 ? 1e300 : 0.0));
      if (g > 0.0) {
        // second-order eigenvalue correction T_ji T_ij / (T_jj - T_ii)
        const cplx tji = Tp[(long long)j * kmax + i];
        corr = cadd(corr, cdiv(cmul(tji, tij), gap));
      }
    }
  }
  off = block_max(off, red);
  eta = block_max(eta, red);
  dmax = block_max(dmax, red);
  if (st == 0) {
    const double scale = fmax(dmax, off);
    const double op = offprev[p];
    // converged at the rounding floor: off-diagonal below 1e-13 of ||T||, or
    // below 1e-11 and no longer shrinking (quadratic steps have stalled)
    const bool conv = off <= 1e-13 * scale || (off <= 1e-11 * scale && off > 0.1 * op);
    // no bound on eta: right after the block step the rotated columns still
    // get their O(1) components along the good ones (exact to first order)
    const bool bad = !(eta < 1e12) || !(scale > 0.0);
    if (bad) st = 2;
    else if (conv) {
      st = 1;
      if (j == 0 && p < 8) g_refine_stats[p] = it;
      if (j < k) lamd[(long long)p * kmax + j] = cadd(d[j], corr);
    } else if (last) st = 2;
  }
  __syncthreads();
  if (j == 0) {
    state[p] = st;
    offprev[p] = off;
  }
  // F: the update of this step (also on the converging step), identity otherwise
  const bool upd = (st_s == 0) && (st != 2);
  if (j < kmax) {
    const cplx dj = d[j];
    for (int i = 0; i < kmax; ++i) {
      cplx f = cmk(0.0, 0.0);
      if (upd && i != j && i < k && j < k) {
        const cplx gap = csub(dj, d[i]);
        if (gap.x != 0.0 || gap.y != 0.0) f = cdiv(Tp[(long long)i * kmax + j], gap);
      }
      const double one = i == j ? 1.0 : 0.0;
      Fp[(long long)i * kmax + j] = cmk(one + f.x, f.y);     // I + F
      Fmp[(long long)i * kmax + j] = cmk(one - f.x, -f.y);   // I - F ~ (I + F)^-1

    }
  }
}

// Sorted (re, im) eigenvalues and unit-norm eigenvector columns in the same
// order; info = -1 for problems that did not converge (the caller falls back).
__global__ void __launch_bounds__(RT) refine_final_kernel(const cplx* __restrict__ W, const cplx* __restrict__ lamd,
                                                          const int* __restrict__ state, const int* __restrict__ kdim,
                                                          int kmax, const int* __restrict__ binfo,
                                                          cplx* __restrict__ lam, cplx* __restrict__ S, long long lds,
                                                          long long sS, int* __restrict__ info) {
  const int p = blockIdx.x, i = threadIdx.x;
  const int k = kdim[p];
  // a singular B~ W0 also goes back to the QR path, which tells a singular B~
  // (IndefiniteBError) from a singular W0
  if (i == 0) info[p] = (binfo[p] == 0 && state[p] == 1) ? 0 : -1;
  if (binfo[p] != 0 || state[p] != 1 || i >= k) return;
  const cplx* lp = lamd + (long long)p * kmax;
  const cplx li = lp[i];
  int rank = 0;
  for (int j = 0; j < k; ++j) {
    const cplx lj = lp[j];
    rank += (lj.x < li.x) || (lj.x == li.x && (lj.y < li.y || (lj.y == li.y && j < i)));
  }
  lam[(long long)p * kmax + rank] = li;
  const cplx* Wp = W + moff(p, kmax);
  double nrm = 0.0;
  for (int r = 0; r < k; ++r) nrm += cabs2(Wp[(long long)r * kmax + i]);
  const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 1.0;
  cplx* Sp = S + (long long)p * sS;
  for (int r = 0; r < kmax; ++r)
    Sp[(long long)r * lds + rank] = r < k ? cscale(Wp[(long long)r * kmax + i], inv) : cmk(0.0, 0.0);
}

struct RefLayout {
  cplx *W, *W2, *Yh, *Yh2, *AW, *BW, *T, *X, *F, *Fm, *LU, *I, *lamd, *Tbb, *Ibb, *Vbb, *lam_b;
  double *offprev, *minpiv;
  int *state, *ipiv, *perm, *winfo, *rhs_of, *nbad, *bad, *kdim_b, *sel_b, *info_b;
  void *gws_b, *scr_b;
};
constexpr int NMATS = 12;

long long small_bytes(int nprob) {
  return (long long)nprob * (3 * KB * KB * 16 + KB * 16 + (3 + 2 * KB) * 4) + 512 +
         (cirr_gen_eig_ws_bytes(KB, nprob) + 255) / 256 * 256 + cirr_gen_eig_vec_scratch_bytes(KB, nprob, KB);
}

RefLayout ref_layout(void* ws, int kmax, int nprob) {
  const long long kk = (long long)kmax * kmax, mats = (long long)nprob * kk;
  RefLayout L;
  cplx* c = reinterpret_cast<cplx*>(ws);
  cplx** m[NMATS] = {&L.W, &L.W2, &L.Yh, &L.Yh2, &L.AW, &L.BW, &L.T, &L.X, &L.F, &L.Fm, &L.LU, &L.I};
  for (int i = 0; i < NMATS; ++i) { *m[i] = c; c += mats; }
  L.lamd = c; c += (long long)nprob * kmax;
  L.Tbb = c; c += (long long)nprob * KB * KB;
  L.Ibb = c; c += (long long)nprob * KB * KB;
  L.Vbb = c; c += (long long)nprob * KB * KB;
  L.lam_b = c; c += (long long)nprob * KB;
  double* d = reinterpret_cast<double*>(c);
  L.offprev = d; d += nprob;
  L.minpiv = d; d += nprob;
  int* q = reinterpret_cast<int*>(d);
  L.state = q; q += nprob;
  L.ipiv = q; q += (long long)nprob * kmax;
  L.perm = q; q += (long long)nprob * kmax;
  L.winfo = q; q += nprob;
  L.rhs_of = q; q += nprob;
  L.nbad = q; q += nprob;
  L.bad = q; q += (long long)nprob * KB;
  L.kdim_b = q; q += nprob;
  L.sel_b = q; q += (long long)nprob * KB;
  L.info_b = q; q += nprob;
  unsigned char* v = reinterpret_cast<unsigned char*>(q);
  v = reinterpret_cast<unsigned char*>(((uintptr_t)v + 255) & ~(uintptr_t)255);
  L.gws_b = v;
  v += (cirr_gen_eig_ws_bytes(KB, nprob) + 255) / 256 * 256;
  L.scr_b = v;
  return L;
}

}  // namespace

CIRR_API long long cirr_gen_eig_refine_ws_bytes(int kmax, int nprob) {
  const long long kk = (long long)kmax * kmax;
  return (long long)nprob * (NMATS * kk * 16 + (long long)kmax * 16 + 16 + 2 * (long long)kmax * 4 + 16) + 1024 +
         small_bytes(nprob);
}

// Eigenpairs of the pencils (A~, B~) (nprob problems, k_b x k_b in a kmax x
// kmax zero-padded block, row-major ld kmax, k <= 256) from approximate
// eigenvectors: W0h[p] (ld ldw, stride sw) holds W0^H, e.g. S^H Q for the
// refinement block S and its orthonormal basis Q.  lam: nprob x kmax sorted by
// (re, im); S[p] (ld lds, stride sS): the unit-norm eigenvectors in that order;
// info: 0 ok, -1 not converged in max_iter steps or B~ W0 exactly singular
// (use the QR path for that problem).
//
// Two-sided form: Yh ~ (B~ W)^-1 is carried along instead of refactoring, so
// one step is seven k x k GEMMs -- T = Yh (A~ W) after a Newton-Schulz
// correction Yh <- (2I - Yh B~ W) Yh, then W <- W (I + F), Yh <- (I - F) Yh.
// The only LU is the one of B~ W0 at the start.
CIRR_API int cirr_gen_eig_refine(const cplx* At, const cplx* Bt, const int* kdim, int kmax, int nprob,
                                 const cplx* W0h, long long ldw, long long sw, int max_iter, void* ws, cplx* lam,
                                 cplx* S, long long lds, long long sS, int* info, cudaStream_t stream) {
  if (kmax <= 0 || kmax > RT || nprob <= 0 || max_iter < 1 || ws == nullptr) return CIRR_EINVAL;
  const long long kk = (long long)kmax * kmax;
  RefLayout L = ref_layout(ws, kmax, nprob);
  cudaError_t e;
  const dim3 fgrid((unsigned)((kk + 255) / 256), nprob);
  auto gemm = [&](const cplx* A, const cplx* B, cplx* C, double alpha, int beta) {
    return cirr_gemm(0, kmax, kmax, kmax, nprob, A, kmax, kk, B, kmax, kk, C, kmax, kk, alpha, beta, stream);
  };
  refine_iota_kernel<<<(nprob + 127) / 128, 128, 0, stream>>>(L.rhs_of, nprob);
  CIRR_CHECK_LAUNCH();
  refine_fill_identity_kernel<<<fgrid, 256, 0, stream>>>(L.I, kdim, kmax, 1.0);
  CIRR_CHECK_LAUNCH();
  refine_init_kernel<<<nprob, RT, 0, stream>>>(W0h, ldw, sw, kdim, kmax, L.W, L.state, L.offprev);
  CIRR_CHECK_LAUNCH();
  // Yh = (B~ W)^-1 (B~'s zero padding meets W's identity padding: B~ W is
  // singular there, so its padding is set to I as well)
  CIRR_TRY(gemm(Bt, L.W, L.LU, 1.0, 0));
  refine_pad_kernel<<<nprob, 128, 0, stream>>>(L.LU, kdim, kmax);
  CIRR_CHECK_LAUNCH();
  CIRR_TRY(cirr_zgetrf_batched(L.LU, kmax, kmax, kk, nprob, L.ipiv, L.perm, L.minpiv, L.winfo, nullptr, stream));
  CIRR_TRY(cirr_zgetrs_batched(L.LU, kmax, kmax, kk, nprob, L.perm, L.I, kmax, kk, L.rhs_of, kmax, L.Yh, kmax, kk,
                               nullptr, stream));
  // T = Yh A~ W; the columns that are not near eigenvectors are replaced from
  // their block's eigenvectors
  CIRR_TRY(gemm(At, L.W, L.AW, 1.0, 0));
  CIRR_TRY(gemm(L.Yh, L.AW, L.T, 1.0, 0));
  refine_classify_kernel<<<nprob, RT, 0, stream>>>(L.T, kdim, kmax, L.state, L.nbad, L.bad, L.Tbb, L.Ibb, L.kdim_b,
                                                   L.sel_b);
  CIRR_CHECK_LAUNCH();
  CIRR_TRY(cirr_gen_eig_values(L.Tbb, nullptr, L.kdim_b, KB, nprob, L.gws_b, L.lam_b, L.info_b, stream));
  CIRR_TRY(cirr_gen_eig_vectors(L.gws_b, L.kdim_b, KB, nprob, L.lam_b, L.sel_b, L.kdim_b, KB, L.scr_b, L.Vbb, KB,
                                (long long)KB * KB, stream));
  refine_rotate_kernel<<<nprob, RT, 0, stream>>>(L.W, L.Yh, kdim, kmax, L.nbad, L.bad, L.Vbb, L.info_b, L.state);
  CIRR_CHECK_LAUNCH();
  cplx *W = L.W, *W2 = L.W2, *Yh = L.Yh, *Yh2 = L.Yh2;
  for (int it = 0; it < max_iter; ++it) {
    CIRR_TRY(gemm(At, W, L.AW, 1.0, 0));
    CIRR_TRY(gemm(Bt, W, L.BW, 1.0, 0));
    // Newton-Schulz: Yh <- (2I - Yh B~ W) Yh (every matrix is block diagonal:
    // the k x k block and the padding, where B~ W = 0, Yh = I and X = I)
    refine_fill_identity_kernel<<<fgrid, 256, 0, stream>>>(L.X, kdim, kmax, 2.0);
    CIRR_CHECK_LAUNCH();
    CIRR_TRY(gemm(Yh, L.BW, L.X, -1.0, 1));
    CIRR_TRY(gemm(L.X, Yh, Yh2, 1.0, 0));
    std::swap(Yh, Yh2);
    CIRR_TRY(gemm(Yh, L.AW, L.T, 1.0, 0));
    refine_update_kernel<<<nprob, RT, 0, stream>>>(L.T, kdim, kmax, L.winfo, L.state, L.offprev, L.F, L.Fm, L.lamd, it,
                                                   it == max_iter - 1 ? 1 : 0);
    CIRR_CHECK_LAUNCH();
    CIRR_TRY(gemm(W, L.F, W2, 1.0, 0));
    std::swap(W, W2);
    CIRR_TRY(gemm(L.Fm, Yh, Yh2, 1.0, 0));
    std::swap(Yh, Yh2);
  }
  refine_final_kernel<<<nprob, RT, 0, stream>>>(W, L.lamd, L.state, kdim, kmax, L.winfo, lam, S, lds, sS, info);
  CIRR_CHECK_LAUNCH();
  (void)e;
  return 0;
}

// debug: g_refine_stats of the last cirr_gen_eig_refine (16 ints: converged
// step of problems 0..7, block-step columns of problems 0..7)
CIRR_API int cirr_gen_eig_refine_stats(int* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_refine_stats, sizeof(int) * 16);
}
