// K4: rank-revealing orthonormalisation of the stacked moment block.
//
// Replaces linalg.py:107-119 (thin SVD of S, keep left singular vectors with
// sigma_i >= rel_tol * sigma_max).  It must resolve sigma ratios near 1e-12:
// config 4's block has sigma_min/sigma_max ~ 2e-12 and a 1e-8 cut loses most
// pairs (finding 7), so Gram-based CholeskyQR is out.
// Algorithm: Householder QR of S (backward stable), one-sided Jacobi SVD of
// the small R with the rotations accumulated (QR preconditioning makes R
// graded: ~3x fewer sweeps than Jacobi on S), then Q = Q_house [U_R; 0] for
// the kept singular vectors.  Jacobi rounds use the circle-method tournament;
// everything runs in one cooperative kernel with a software grid barrier
// between dependent steps; all reductions are fixed-order (bit-reproducible).
#include "common.cuh"
#include <cstdlib>
#include "cirr.h"

namespace {

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
constexpr int JB_MAX = 8;   // rows per Jacobi block (fewer for wide blocks: 4 * jb rows of length c in smem)
__device__ long long g_orth_phase[4];
#define ORTH_MARK(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_orth_phase[i] = clock64(); } while (0)

// One Householder step of the QR of S (rows of W are the columns of S): the
// reflector of column j (one CTA per problem), then H_j^H applied to columns
// j+1 .. qend-1 (one CTA per problem x column), a grid barrier after each.
__device__ void householder_step(cplx* __restrict__ W, long long ldw, long long wstride, int n, int c, int nprob,
                                 int j, int qend, cplx* __restrict__ tau, unsigned* bar, double (*red)[HT / 32],
                                 double* sred) {
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int p = blockIdx.x; p < nprob; p += G) {
    cplx* x = W + (long long)p * wstride + (long long)j * ldw;
    double sq = 0.0;
    for (int i = j + 1 + tid; i < n; i += HT) sq += cabs2(x[i]);
    sq = block_sum(sq, sred);
    const cplx alpha = x[j];
    cplx t = cmk(0.0, 0.0);
    if (sq != 0.0 || alpha.y != 0.0) {
      double beta = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + sq);
      beta = alpha.x >= 0.0 ? -beta : beta;
      t = cmk((beta - alpha.x) / beta, -alpha.y / beta);
      const cplx scal = crecip(cmk(alpha.x - beta, alpha.y));
      for (int i = j + 1 + tid; i < n; i += HT) x[i] = cmul(x[i], scal);
      __syncthreads();
      if (tid == 0) x[j] = cmk(beta, 0.0);
    }
    if (tid == 0) tau[(long long)p * c + j] = t;
  }
  grid_barrier(bar, G);
  const int rest = qend - j - 1;
  const long long items = (long long)nprob * (rest > 0 ? rest : 0);
  for (long long it = blockIdx.x; it < items; it += G) {
    const int p = (int)(it / rest), q = j + 1 + (int)(it % rest);
    const cplx t = tau[(long long)p * c + j];
    if (t.x == 0.0 && t.y == 0.0) continue;
    const cplx* v = W + (long long)p * wstride + (long long)j * ldw;
    cplx* y = W + (long long)p * wstride + (long long)q * ldw;
    double wr = 0.0, wi = 0.0;
    for (int i = j + tid; i < n; i += HT) {
      const cplx vi = i == j ? cmk(1.0, 0.0) : v[i];
      const cplx g = cconjmul(vi, y[i]);
      wr += g.x;
      wi += g.y;
    }
    wr = warp_sum(wr); wi = warp_sum(wi);
    __syncthreads();
    if (lane == 0) { red[0][wid] = wr; red[1][wid] = wi; }
    __syncthreads();
    wr = 0.0; wi = 0.0;
    for (int w2 = 0; w2 < HT / 32; ++w2) { wr += red[0][w2]; wi += red[1][w2]; }
    const cplx f = cmul(cconj(t), cmk(wr, wi));
    for (int i = j + tid; i < n; i += HT) {
      const cplx vi = i == j ? cmk(1.0, 0.0) : v[i];
      cfms(y[i], vi, f);
    }
  }
  grid_barrier(bar, G);
}

// Panel of the blocked QR: Householder steps j0 .. j1-1, each applied only to
// the panel's own later columns (the rest of S gets the block as WY products).
__global__ void __launch_bounds__(HT) qr_panel_kernel(cplx* __restrict__ W, long long ldw, long long wstride, int n,
                                                      int c, int nprob, int j0, int j1, cplx* __restrict__ tau,
                                                      unsigned* bar) {
  __shared__ double red[4][HT / 32];
  __shared__ double sred[32];
  for (int j = j0; j < j1; ++j) householder_step(W, ldw, wstride, n, c, nprob, j, j1, tau, bar, red, sred);
}

// --------------------------------------------------------------------------
// QR-preconditioned one-sided Jacobi (the production path).
//
//  A. Householder QR of S (n x c): the columns of S are the rows of W, so every
//     reflector and every update works on contiguous rows.  Reflector j is
//     stored in row j of W below the diagonal (LAPACK layout) with R above it.
//  B. One-sided Jacobi on the rows of R (length c) with the rotations
//     accumulated into J: R^H J = X Sigma  =>  R = J Sigma X^H, so J holds the
//     left singular vectors of R.  R after QR is graded, which cuts the sweep
//     count ~3x against Jacobi on S itself (Drmac-Veselic preconditioning),
//     and each rotation touches c instead of n entries.
//  C. sigma = row norms, descending sort, rank cut; Q = H_0 ... H_{c-1} [J_kept; 0].
// One cooperative launch; grid barriers separate the dependent steps.
__global__ void __launch_bounds__(HT) qr_jacobi_kernel(cplx* __restrict__ W, long long ldw, long long wstride,
                                                        int n, int c, int nprob, double rel_tol,
                                                        double* __restrict__ sigma, int* __restrict__ order,
                                                        int* __restrict__ kept, cplx* __restrict__ Qt,
                                                        long long ldq, long long qstride, unsigned* bar,
                                                        int* counters, cplx* __restrict__ Xc,
                                                        cplx* __restrict__ Jt, cplx* __restrict__ tau,
                                                        int max_sweeps, double tol, int* sweeps_out, int JB,
                                                        int back, int do_qr) {
  __shared__ double red[4][HT / 32];
  __shared__ double sred[32];
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int jmax = min(c, n);
  const long long cc = (long long)c * c;
  ORTH_MARK(0);
  // ---------------- A: Householder QR ----------------
  if (do_qr)
    for (int j = 0; j < jmax; ++j) householder_step(W, ldw, wstride, n, c, nprob, j, c, tau, bar, red, sred);
  ORTH_MARK(1);
  // ---------------- B: Jacobi on the rows of R ----------------
  // Xc[p][a][i] = conj(R[a][i]) (R[a][i] = W[p][i][a] for a <= i < c, a < jmax), Jt = I
  {
    const long long total = (long long)nprob * cc;
    for (long long e = (long long)blockIdx.x * HT + tid; e < total; e += (long long)G * HT) {
      const int p = (int)(e / cc);
      const int a = (int)((e % cc) / c), i = (int)(e % c);
      const cplx r = (a <= i && a < jmax) ? W[(long long)p * wstride + (long long)i * ldw + a] : cmk(0.0, 0.0);
      Xc[e] = cconj(r);
      Jt[e] = cmk(a == i ? 1.0 : 0.0, 0.0);
    }
  }
  if (blockIdx.x == 0 && tid == 0) { counters[0] = 0; counters[1] = 0; }
  grid_barrier(bar, G);
  // block-cyclic one-sided Jacobi: rows are grouped in blocks of JB; each outer
  // round pairs blocks (circle method) and a CTA rotates every row pair of its
  // 2*JB rows in shared memory (one local sweep), so the grid synchronises once
  // per block round instead of once per row round.
  extern __shared__ __align__(16) cplx jsm[];
  cplx* sx = jsm;                       // 2*JB rows of Xc (length c)
  cplx* sj = jsm + 2 * JB * (long long)c; // 2*JB rows of Jt
  __shared__ int s_rot;
  const int nblk = (c + JB - 1) / JB;
  const int bp = nblk + (nblk & 1);
  const int npairs = bp / 2;
  const long long pitems = (long long)nprob * npairs;
  int sweep = 0;
  for (; sweep < max_sweeps && c > 1; ++sweep) {
    if (blockIdx.x == 0 && tid == 0) counters[(sweep + 1) & 1] = 0;
    for (int round = 0; round < max(bp - 1, 1); ++round) {
      for (long long it = blockIdx.x; it < pitems; it += G) {
        const int p = (int)(it / npairs), kk = (int)(it % npairs);
        int bI, bJ;
        if (nblk == 1) { bI = 0; bJ = bp; }  // single block: local sweep only
        else rr_pair(round, kk, bp, bI, bJ);
        if (bI >= nblk && bJ >= nblk) continue;
        if (bI >= nblk) { bI = bJ; bJ = nblk; }
        // local rows: block I then block J (J may be absent)
        const int r0 = bI * JB, n0 = min(JB, c - r0);
        const int r1 = bJ < nblk ? bJ * JB : 0, n1 = bJ < nblk ? min(JB, c - r1) : 0;
        const int nl = n0 + n1;
        cplx* Xp = Xc + (long long)p * cc;
        cplx* Jp = Jt + (long long)p * cc;
        for (int e = tid; e < nl * c; e += HT) {
          const int lr = e / c, i = e % c;
          const int gr = lr < n0 ? r0 + lr : r1 + lr - n0;
          sx[(long long)lr * c + i] = Xp[(long long)gr * c + i];
          sj[(long long)lr * c + i] = Jp[(long long)gr * c + i];
        }
        if (tid == 0) s_rot = 0;
        __syncthreads();
        // one local sweep over all pairs of the nl rows (circle method, a warp per pair)
        const int lp = nl + (nl & 1);
        for (int lround = 0; lround < lp - 1; ++lround) {
          for (int pk = wid; pk < lp / 2; pk += HT / 32) {
            int a, b2;
            rr_pair(lround, pk, lp, a, b2);
            if (a >= nl || b2 >= nl) continue;
            if (a > b2) { int t = a; a = b2; b2 = t; }
            cplx* xa = sx + (long long)a * c;
            cplx* xb = sx + (long long)b2 * c;
            double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
            for (int i = lane; i < c; i += 32) {
              const cplx x = xa[i], y = xb[i];
              al += cabs2(x);
              be += cabs2(y);
              const cplx g = cconjmul(x, y);
              gr += g.x;
              gi += g.y;
            }
            al = warp_sum(al); be = warp_sum(be); gr = warp_sum(gr); gi = warp_sum(gi);
            const double ag = hypot(gr, gi);
            if (al > 0.0 && be > 0.0 && ag > tol * sqrt(al) * sqrt(be)) {
              const double zeta = (be - al) / (2.0 * ag);
              const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
              const double cs = 1.0 / sqrt(1.0 + t * t), sn = t * cs;
              const cplx se = cmk(sn * gr / ag, sn * gi / ag);
              const cplx sec = cconj(se);
              cplx* ja = sj + (long long)a * c;
              cplx* jb = sj + (long long)b2 * c;
              for (int i = lane; i < c; i += 32) {
                const cplx x = xa[i], y = xb[i];
                xa[i] = csub(cscale(x, cs), cmul(sec, y));
                xb[i] = cadd(cmul(se, x), cscale(y, cs));
                const cplx u = ja[i], w = jb[i];
                ja[i] = csub(cscale(u, cs), cmul(sec, w));
                jb[i] = cadd(cmul(se, u), cscale(w, cs));
              }
              if (lane == 0) atomicAdd(&s_rot, 1);
            }
          }
          __syncthreads();
        }
        for (int e = tid; e < nl * c; e += HT) {
          const int lr = e / c, i = e % c;
          const int gr = lr < n0 ? r0 + lr : r1 + lr - n0;
          Xp[(long long)gr * c + i] = sx[(long long)lr * c + i];
          Jp[(long long)gr * c + i] = sj[(long long)lr * c + i];
        }
        if (tid == 0 && s_rot > 0) atomicAdd(counters + (sweep & 1), s_rot);
        __syncthreads();
      }
      grid_barrier(bar, G);
    }
    const int rots = *((volatile int*)(counters + (sweep & 1)));
    grid_barrier(bar, G);
    if (rots == 0) { ++sweep; break; }
  }
  if (blockIdx.x == 0 && tid == 0) *sweeps_out = sweep;
  ORTH_MARK(2);
  // ---------------- C: singular values, rank cut, Q ----------------
  for (int p = blockIdx.x; p < nprob; p += G) {
    double* sg = reinterpret_cast<double*>(tau + (long long)nprob * c) + (long long)p * c;  // scratch
    for (int a = wid; a < c; a += HT / 32) {
      double s2 = 0.0;
      for (int i = lane; i < c; i += 32) s2 += cabs2(Xc[(long long)p * cc + (long long)a * c + i]);
      s2 = warp_sum(s2);
      if (lane == 0) sg[a] = sqrt(s2);
    }
    __syncthreads();
    double smax = 0.0;
    for (int a = 0; a < c; ++a) smax = fmax(smax, sg[a]);
    for (int a = tid; a < c; a += HT) {
      const double sa = sg[a];
      int rank = 0;
      for (int b3 = 0; b3 < c; ++b3) {
        const double sb = sg[b3];
        rank += (sb > sa) || (sb == sa && b3 < a);
      }
      order[(long long)p * c + rank] = a;
      sigma[(long long)p * c + rank] = sa;
    }
    if (tid == 0) {
      int k = 0;
      if (smax > 0.0)
        for (int a = 0; a < c; ++a) k += sg[a] >= rel_tol * smax;
      kept[p] = k;
    }
    __syncthreads();
  }
  if (!back) return;  // C runs as blocked (WY) GEMMs after this kernel (orth_back_blocked)
  grid_barrier(bar, G);
  // Qt[p][r] = [J[:, order[r]]; 0] for r < kept[p]
  for (long long e = (long long)blockIdx.x * HT + tid; e < (long long)nprob * c * n; e += (long long)G * HT) {
    const int p = (int)(e / ((long long)c * n));
    const int r = (int)((e / n) % c), i = (int)(e % n);
    if (r >= kept[p]) continue;
    const int a = order[(long long)p * c + r];
    Qt[(long long)p * qstride + (long long)r * ldq + i] = i < c ? Jt[(long long)p * cc + (long long)a * c + i]
                                                              : cmk(0.0, 0.0);
  }
  grid_barrier(bar, G);
  // apply H_{jmax-1}, ..., H_0 to every kept row of Qt (a column of Q)
  for (int j = jmax - 1; j >= 0; --j) {
    const long long items = (long long)nprob * c;
    for (long long it = blockIdx.x; it < items; it += G) {
      const int p = (int)(it / c), r = (int)(it % c);
      if (r >= kept[p]) continue;
      const cplx t = tau[(long long)p * c + j];
      if (t.x == 0.0 && t.y == 0.0) continue;
      const cplx* v = W + (long long)p * wstride + (long long)j * ldw;
      cplx* y = Qt + (long long)p * qstride + (long long)r * ldq;
      double wr = 0.0, wi = 0.0;
      for (int i = j + tid; i < n; i += HT) {
        const cplx vi = i == j ? cmk(1.0, 0.0) : v[i];
        const cplx g = cconjmul(vi, y[i]);
        wr += g.x;
        wi += g.y;
      }
      wr = warp_sum(wr); wi = warp_sum(wi);
      __syncthreads();
      if (lane == 0) { red[0][wid] = wr; red[1][wid] = wi; }
      __syncthreads();
      wr = 0.0; wi = 0.0;
      for (int w2 = 0; w2 < HT / 32; ++w2) { wr += red[0][w2]; wi += red[1][w2]; }
      const cplx f = cmul(t, cmk(wr, wi));
      for (int i = j + tid; i < n; i += HT) {
        const cplx vi = i == j ? cmk(1.0, 0.0) : v[i];
        cfms(y[i], vi, f);
      }
    }
    grid_barrier(bar, G);
  }
  ORTH_MARK(3);
}

}  // namespace

namespace {
constexpr int WYB = 32;  // reflectors per WY block

// W[p] (c x n, row j = reflector j below its diagonal, R on and above it) ->
// V^T in place: zeros before the diagonal, the implicit unit on it.
__global__ void wy_prep_kernel(cplx* __restrict__ W, long long ldw, long long wstride, int n, int c) {
  const int p = blockIdx.z, j = blockIdx.y;
  cplx* row = W + (long long)p * wstride + (long long)j * ldw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= j && i < n; i += gridDim.x * blockDim.x)
    row[i] = cmk(i == j ? 1.0 : 0.0, 0.0);
}

// X[p] (n x c, row-major): X[i][r] = J[i][order[r]] for i < c and r < kept[p], else 0.
__global__ void wy_init_x_kernel(const cplx* __restrict__ Jt, const int* __restrict__ order,
                                 const int* __restrict__ kept, int n, int c, cplx* __restrict__ X) {
  const int p = blockIdx.z, i = blockIdx.y;
  const long long cc = (long long)c * c;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < c; r += gridDim.x * blockDim.x) {
    cplx v = cmk(0.0, 0.0);
    if (i < c && r < kept[p]) v = Jt[(long long)p * cc + (long long)order[(long long)p * c + r] * c + i];
    X[(long long)p * n * c + (long long)i * c + r] = v;
  }
}

// T of one block (LAPACK larft, forward, columnwise): T[i][i] = tau_i,
// T[0:i, i] = -tau_i T[0:i, 0:i] G[0:i, i] with G = V^H V (WYB x WYB).
__global__ void wy_tfac_kernel(const cplx* __restrict__ Gm, const cplx* __restrict__ tau, int c, int j0, int nb,
                               cplx* __restrict__ T) {
  const int p = blockIdx.x, t = threadIdx.x;
  const cplx* G = Gm + (long long)p * WYB * WYB;
  const cplx* tp = tau + (long long)p * c + j0;
  __shared__ cplx sT[WYB][WYB + 1];
  for (int e = t; e < WYB * WYB; e += blockDim.x) sT[e / WYB][e % WYB] = cmk(0.0, 0.0);
  __syncthreads();
  for (int i = 0; i < nb; ++i) {
    const cplx ti = tp[i];
    cplx acc = cmk(0.0, 0.0);
    if (t < i)
      for (int l = t; l < i; ++l) cfma(acc, sT[t][l], G[(long long)l * WYB + i]);
    __syncthreads();
    if (t < i) sT[t][i] = cmul(cmk(-ti.x, -ti.y), acc);
    if (t == i) sT[i][i] = ti;
    __syncthreads();
  }
  cplx* Tp = T + (long long)p * WYB * WYB;
  for (int e = t; e < WYB * WYB; e += blockDim.x) Tp[e] = sT[e / WYB][e % WYB];
}
}  // namespace

namespace {
// Panel j0 .. j0+nb-1 of the blocked QR as explicit reflectors: VT[p] (WYB x n,
// row m = v_{j0+m}: zeros before j0+m, 1 on it) and Vn[p] = VT[p]^T (n x WYB).
__global__ void qr_panel_v_kernel(const cplx* __restrict__ W, long long ldw, long long wstride, int n, int j0, int nb,
                                  cplx* __restrict__ VT, cplx* __restrict__ Vn) {
  const int p = blockIdx.z, m = blockIdx.y;
  const int j = j0 + m;
  const cplx* row = W + (long long)p * wstride + (long long)j * ldw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const cplx v = m >= nb ? cmk(0.0, 0.0) : (i < j ? cmk(0.0, 0.0) : (i == j ? cmk(1.0, 0.0) : row[i]));
    VT[(long long)p * WYB * n + (long long)m * n + i] = v;
    Vn[(long long)p * n * WYB + (long long)i * WYB + m] = v;
  }
}
}  // namespace

// Phase A of cirr_orth blocked: panels of WYB columns factored by
// qr_panel_kernel (cooperative, one CTA per problem x column), the rest of S
// updated per panel as S_t -= V (T^H (V^H S_t)) on the batched GEMM.  In the
// row layout of W (S_t^T = W_t, rest x n) the three products are
// Q1 = conj(W_t) V (= conj(V^H S_t)^T), Q2 = Q1 T, W_t -= conj(Q2) V^T.
// The per-column grid-wide pass over all later columns (~100 us per column
// at n = 8000, c = 256, 4 problems) shrinks to the panel's own columns.
static int orth_qr_blocked(cplx* W, long long ldw, long long wstride, int n, int c, int nprob, cplx* tau,
                           unsigned* bar, int cap, cudaStream_t stream) {
  const int jmax = c < n ? c : n;
  cplx *VT = nullptr, *Vn = nullptr, *Gm = nullptr, *Q1 = nullptr;
  const size_t nv = (size_t)n * WYB * nprob;
  cudaError_t e = cirr_malloc_async(reinterpret_cast<void**>(&VT), sizeof(cplx) * 2 * nv, stream);
  if (e == cudaSuccess)
    e = cirr_malloc_async(reinterpret_cast<void**>(&Gm), sizeof(cplx) * (size_t)2 * WYB * WYB * nprob, stream);
  if (e == cudaSuccess)
    e = cirr_malloc_async(reinterpret_cast<void**>(&Q1), sizeof(cplx) * (size_t)2 * WYB * c * nprob, stream);
  if (e != cudaSuccess) {
    for (cplx* q : {VT, Gm}) if (q) cudaFreeAsync(q, stream);
    return (int)e;
  }
  Vn = VT + nv;
  cplx* T = Gm + (size_t)WYB * WYB * nprob;
  cplx* Q2 = Q1 + (size_t)WYB * c * nprob;
  const long long sv = (long long)n * WYB, sq = (long long)c * WYB, st = (long long)WYB * WYB;
  int rc = 0;
  for (int j0 = 0; rc == 0 && j0 < jmax; j0 += WYB) {
    const int nb = (jmax - j0) < WYB ? (jmax - j0) : WYB;
    const int j1 = j0 + nb;
    long long want = (long long)nprob * nb;
    int grid = (int)(want < cap ? want : cap);
    int j0v = j0, j1v = j1;
    void* args[] = {&W, &ldw, &wstride, &n, &c, &nprob, &j0v, &j1v, &tau, &bar};
    rc = (int)cudaLaunchCooperativeKernel((void*)qr_panel_kernel, dim3(grid), dim3(HT), args, 0, stream);
    cirr_note_launch();
    const int rest = c - j1;
    if (rc || rest <= 0) continue;
    {
      dim3 g((n + 255) / 256, WYB, nprob);
      qr_panel_v_kernel<<<g, 256, 0, stream>>>(W, ldw, wstride, n, j0, nb, VT, Vn);
      rc = (int)cudaGetLastError();
      cirr_note_launch();
      if (rc) break;
    }
    // G = V^H V, T (larft)
    rc = cirr_gemm(1, nb, nb, n, nprob, VT, n, sv, Vn, WYB, sv, Gm, WYB, st, 1.0, 0, stream);
    if (rc) break;
    wy_tfac_kernel<<<nprob, WYB, 0, stream>>>(Gm, tau, c, j0, nb, T);
    rc = (int)cudaGetLastError();
    cirr_note_launch();
    if (rc) break;
    cplx* Wt = W + (long long)j1 * ldw;
    rc = cirr_gemm(1, rest, WYB, n, nprob, Wt, ldw, wstride, Vn, WYB, sv, Q1, WYB, sq, 1.0, 0, stream);
    if (rc) break;
    rc = cirr_gemm(0, rest, WYB, WYB, nprob, Q1, WYB, sq, T, WYB, st, Q2, WYB, sq, 1.0, 0, stream);
    if (rc) break;
    rc = cirr_gemm(1, rest, n, WYB, nprob, Q2, WYB, sq, VT, n, sv, Wt, ldw, wstride, -1.0, 1, stream);
  }
  cudaFreeAsync(VT, stream);
  cudaFreeAsync(Gm, stream);
  cudaFreeAsync(Q1, stream);
  return rc;
}

// Phase C of cirr_orth as Level-3 products: with V^T = the reflector rows of W
// (unit diagonal, zeros before it) and X = [J_kept; 0] (n x c), apply the WY
// blocks from the last to the first, X -= V (T (V^H X)), then Qt = X^T.
static int orth_back_blocked(cplx* W, long long ldw, long long wstride, int n, int c, int nprob, const int* kept,
                             const int* order, const cplx* Jt, const cplx* tau, cplx* Qt, long long ldq,
                             long long qstride, cudaStream_t stream) {
  const int jmax = c < n ? c : n;
  {
    dim3 g(1, c, nprob);
    wy_prep_kernel<<<g, 256, 0, stream>>>(W, ldw, wstride, n, c);
    CIRR_CHECK_LAUNCH();
  }
  cplx *VT = nullptr, *X = nullptr, *Gm = nullptr, *T = nullptr, *Wk = nullptr, *Wk2 = nullptr;
  const size_t nc = (size_t)n * c * nprob;
  cudaError_t e = cirr_malloc_async(reinterpret_cast<void**>(&VT), sizeof(cplx) * nc, stream);
  if (e == cudaSuccess) e = cirr_malloc_async(reinterpret_cast<void**>(&X), sizeof(cplx) * nc, stream);
  if (e == cudaSuccess)
    e = cirr_malloc_async(reinterpret_cast<void**>(&Gm), sizeof(cplx) * (size_t)2 * WYB * WYB * nprob, stream);
  if (e == cudaSuccess)
    e = cirr_malloc_async(reinterpret_cast<void**>(&Wk), sizeof(cplx) * (size_t)2 * WYB * c * nprob, stream);
  if (e != cudaSuccess) {
    for (cplx* q : {VT, X, Gm}) if (q) cudaFreeAsync(q, stream);
    return (int)e;
  }
  T = Gm + (size_t)WYB * WYB * nprob;
  Wk2 = Wk + (size_t)WYB * c * nprob;
  const long long sv = (long long)n * c;
  int rc = cirr_transpose(0, W, ldw, wstride, c, n, nprob, VT, c, sv, stream);   // V (n x c)
  if (rc == 0) {
    dim3 g((c + 127) / 128, n, nprob);
    wy_init_x_kernel<<<g, 128, 0, stream>>>(Jt, order, kept, n, c, X);
    rc = (int)cudaGetLastError();
    cirr_note_launch();
  }
  const int nblk = (jmax + WYB - 1) / WYB;
  for (int b = nblk - 1; rc == 0 && b >= 0; --b) {
    const int j0 = b * WYB, nb = (jmax - j0) < WYB ? (jmax - j0) : WYB;
    const cplx* Vh = W + (long long)j0 * ldw;   // rows j0.. of V^T (conj -> V^H)
    // G = V^H V, T (larft)
    rc = cirr_gemm(1, nb, nb, n, nprob, Vh, ldw, wstride, VT + j0, c, sv, Gm, WYB, WYB * WYB, 1.0, 0, stream);
    if (rc) break;
    wy_tfac_kernel<<<nprob, WYB, 0, stream>>>(Gm, tau, c, j0, nb, T);
    rc = (int)cudaGetLastError();
    cirr_note_launch();
    if (rc) break;
    // X -= V (T (V^H X))
    rc = cirr_gemm(1, nb, c, n, nprob, Vh, ldw, wstride, X, c, sv, Wk, c, (long long)WYB * c, 1.0, 0, stream);
    if (rc) break;
    rc = cirr_gemm(0, nb, c, nb, nprob, T, WYB, WYB * WYB, Wk, c, (long long)WYB * c, Wk2, c, (long long)WYB * c,
                   1.0, 0, stream);
    if (rc) break;
    rc = cirr_gemm(0, n, c, nb, nprob, VT + j0, c, sv, Wk2, c, (long long)WYB * c, X, c, sv, -1.0, 1, stream);
  }
  if (rc == 0) rc = cirr_transpose(0, X, c, sv, n, c, nprob, Qt, ldq, qstride, stream);
  cudaFreeAsync(VT, stream);
  cudaFreeAsync(X, stream);
  cudaFreeAsync(Gm, stream);
  cudaFreeAsync(Wk, stream);
  return rc;
}

// --------------------------------------------------------------------------
// The same three phases for many small blocks (config 2: 512 blocks of
// n = 256, c = 32): one CTA per problem with the whole block in shared memory,
// so no grid barrier is needed (the cooperative kernel spends ~130 of them per
// call and runs 2.2 ms per 256-block batch there).  Householder QR with a warp
// per trailing row, one-sided Jacobi on the rows of R (circle method over all
// c rows, a warp per pair, same rotation formulas and threshold), sort and
// rank cut, and Q = H_0 ... H_{c-1} [J_kept; 0] with each kept column in the
// registers of one warp.  Results equal the cooperative kernel's to rounding
// (the Jacobi pair order differs).
constexpr int OS_T = 256;
constexpr int OS_NMAX = 512;          // y[OS_NMAX / 32] per lane in phase C
__host__ __device__ constexpr long long orth_small_smem(int n, int c) {
  return (long long)c * n * 16 + 2LL * c * c * 16 + (long long)c * 16 + (long long)c * 8 + (long long)c * 4 + 64;
}

__global__ void __launch_bounds__(OS_T) orth_small_kernel(cplx* __restrict__ W, long long ldw, long long wstride,
                                                          int n, int c, double rel_tol, double* __restrict__ sigma,
                                                          int* __restrict__ order, int* __restrict__ kept,
                                                          cplx* __restrict__ Qt, long long ldq, long long qstride,
                                                          int max_sweeps, double tol, int* __restrict__ sweeps_out) {
  extern __shared__ __align__(16) cplx osm[];
  cplx* A = osm;                                   // c x n: the columns of S as rows, then reflectors / R
  cplx* X = A + (long long)c * n;                  // c x c
  cplx* J = X + (long long)c * c;                  // c x c
  cplx* tau = J + (long long)c * c;                // c
  double* sg = reinterpret_cast<double*>(tau + c); // c
  int* ord = reinterpret_cast<int*>(sg + c);       // c
  __shared__ double sred[32];
  __shared__ int s_rot;
  constexpr int NW = OS_T / 32;
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const cplx* Wp = W + (long long)p * wstride;
  for (int e = tid; e < c * n; e += OS_T) {
    const int r = e / n, i = e - r * n;
    A[e] = Wp[(long long)r * ldw + i];
  }
  __syncthreads();
  const int jmax = min(c, n);
  // ---- A: Householder QR of S (reflector j in row j of A, R above) ----
  for (int j = 0; j < jmax; ++j) {
    cplx* x = A + (long long)j * n;
    double sq = 0.0;
    for (int i = j + 1 + tid; i < n; i += OS_T) sq += cabs2(x[i]);
    sq = block_sum(sq, sred);
    const cplx alpha = x[j];
    cplx t = cmk(0.0, 0.0);
    if (sq != 0.0 || alpha.y != 0.0) {
      double beta = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + sq);
      beta = alpha.x >= 0.0 ? -beta : beta;
      t = cmk((beta - alpha.x) / beta, -alpha.y / beta);
      const cplx scal = crecip(cmk(alpha.x - beta, alpha.y));
      for (int i = j + 1 + tid; i < n; i += OS_T) x[i] = cmul(x[i], scal);
    }
    __syncthreads();
    if (tid == 0) {
      if (sq != 0.0 || alpha.y != 0.0) x[j] = cmk(alpha.x >= 0.0 ? -sqrt(alpha.x * alpha.x + alpha.y * alpha.y + sq)
                                                                 : sqrt(alpha.x * alpha.x + alpha.y * alpha.y + sq),
                                                  0.0);
      tau[j] = t;
    }
    if (t.x != 0.0 || t.y != 0.0) {
      const cplx tc = cconj(t);
      for (int q = j + 1 + wid; q < c; q += NW) {
        cplx* y = A + (long long)q * n;
        double wr = 0.0, wi = 0.0;
        for (int i = j + lane; i < n; i += 32) {
          const cplx vi = i == j ? cmk(1.0, 0.0) : x[i];
          const cplx g = cconjmul(vi, y[i]);
          wr += g.x;
          wi += g.y;
        }
        wr = warp_sum(wr);
        wi = warp_sum(wi);
        const cplx f = cmul(tc, cmk(wr, wi));
        for (int i = j + lane; i < n; i += 32) {
          const cplx vi = i == j ? cmk(1.0, 0.0) : x[i];
          cfms(y[i], vi, f);
        }
      }
    }
    __syncthreads();
  }
  // ---- B: one-sided Jacobi on the rows of X = R^H, rotations into J ----
  for (int e = tid; e < c * c; e += OS_T) {
    const int a = e / c, i = e - a * c;
    X[e] = (a <= i && a < jmax) ? cconj(A[(long long)i * n + a]) : cmk(0.0, 0.0);
    J[e] = cmk(a == i ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  const int lp = c + (c & 1);
  int sweep = 0;
  for (; sweep < max_sweeps && c > 1; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < lp - 1; ++round) {
      for (int pk = wid; pk < lp / 2; pk += NW) {
        int a, b2;
        rr_pair(round, pk, lp, a, b2);
        if (a >= c || b2 >= c) continue;
        if (a > b2) { const int tt = a; a = b2; b2 = tt; }
        cplx* xa = X + (long long)a * c;
        cplx* xb = X + (long long)b2 * c;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        for (int i = lane; i < c; i += 32) {
          const cplx x = xa[i], y = xb[i];
          al += cabs2(x);
          be += cabs2(y);
          const cplx g = cconjmul(x, y);
          gr += g.x;
          gi += g.y;
        }
        al = warp_sum(al); be = warp_sum(be); gr = warp_sum(gr); gi = warp_sum(gi);
        const double ag = hypot(gr, gi);
        if (al > 0.0 && be > 0.0 && ag > tol * sqrt(al) * sqrt(be)) {
          const double zeta = (be - al) / (2.0 * ag);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = t * cs;
          const cplx se = cmk(sn * gr / ag, sn * gi / ag);
          const cplx sec = cconj(se);
          cplx* ja = J + (long long)a * c;
          cplx* jb = J + (long long)b2 * c;
          for (int i = lane; i < c; i += 32) {
            const cplx x = xa[i], y = xb[i];
            xa[i] = csub(cscale(x, cs), cmul(sec, y));
            xb[i] = cadd(cmul(se, x), cscale(y, cs));
            const cplx u = ja[i], w = jb[i];
            ja[i] = csub(cscale(u, cs), cmul(sec, w));
            jb[i] = cadd(cmul(se, u), cscale(w, cs));
          }
          if (lane == 0) atomicAdd(&s_rot, 1);
        }
      }
      __syncthreads();
    }
    if (s_rot == 0) { ++sweep; break; }
    __syncthreads();
  }
  if (tid == 0) atomicMax(sweeps_out, sweep);
  // ---- C: sigma, descending order, rank cut, Q ----
  for (int a = wid; a < c; a += NW) {
    double s2 = 0.0;
    for (int i = lane; i < c; i += 32) s2 += cabs2(X[(long long)a * c + i]);
    s2 = warp_sum(s2);
    if (lane == 0) sg[a] = sqrt(s2);
  }
  __syncthreads();
  double smax = 0.0;
  for (int a = 0; a < c; ++a) smax = fmax(smax, sg[a]);
  for (int a = tid; a < c; a += OS_T) {
    const double sa = sg[a];
    int rank = 0;
    for (int b3 = 0; b3 < c; ++b3) {
      const double sb = sg[b3];
      rank += (sb > sa) || (sb == sa && b3 < a);
    }
    ord[rank] = a;
    order[(long long)p * c + rank] = a;
    sigma[(long long)p * c + rank] = sa;
  }
  int k = 0;
  if (smax > 0.0)
    for (int a = 0; a < c; ++a) k += sg[a] >= rel_tol * smax;
  if (tid == 0) kept[p] = k;
  __syncthreads();
  constexpr int NY = OS_NMAX / 32;
  for (int r = wid; r < k; r += NW) {
    const int a = ord[r];
    cplx y[NY];
#pragma unroll
    for (int s2 = 0; s2 < NY; ++s2) {
      const int i = lane + 32 * s2;
      y[s2] = (i < c && i < n) ? J[(long long)a * c + i] : cmk(0.0, 0.0);
    }
    for (int j = jmax - 1; j >= 0; --j) {
      const cplx t = tau[j];
      if (t.x == 0.0 && t.y == 0.0) continue;
      const cplx* v = A + (long long)j * n;
      double wr = 0.0, wi = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < NY; ++s2) {
        const int i = lane + 32 * s2;
        if (i >= j && i < n) {
          const cplx vi = i == j ? cmk(1.0, 0.0) : v[i];
          const cplx g = cconjmul(vi, y[s2]);
          wr += g.x;
          wi += g.y;
        }
      }
      wr = warp_sum(wr);
      wi = warp_sum(wi);
      const cplx f = cmul(t, cmk(wr, wi));
#pragma unroll
      for (int s2 = 0; s2 < NY; ++s2) {
        const int i = lane + 32 * s2;
        if (i >= j && i < n) {
          const cplx vi = i == j ? cmk(1.0, 0.0) : v[i];
          cfms(y[s2], vi, f);
        }
      }
    }
    cplx* q = Qt + (long long)p * qstride + (long long)r * ldq;
#pragma unroll
    for (int s2 = 0; s2 < NY; ++s2) {
      const int i = lane + 32 * s2;
      if (i < n) q[i] = y[s2];
    }
  }
}

// Workspace bytes for cirr_orth (barrier/counters, X and J (nprob x c x c),
// tau and sigma scratch).
CIRR_API long long cirr_orth_ws_bytes(int c, int nprob) {
  return 4096 + 2LL * nprob * c * c * 16 + (long long)nprob * c * 16 + (long long)nprob * c * 8 + 256;
}

// Rank-revealing orthonormal basis of S (n x c) for nprob blocks; W[prob] holds
// the columns of S as rows (c x n, overwritten by the QR reflectors).
// Outputs: sigma (nprob x c, descending), order (nprob x c), kept (nprob,
// sigma >= rel_tol * sigma_max), Qt[prob] (kept x n rows: orthonormal columns
// of Q spanning the kept left singular vectors).  ws: cirr_orth_ws_bytes.
// *sweeps_out (device int) = Jacobi sweeps used.
CIRR_API int cirr_orth(cplx* W, long long ldw, long long wstride, int n, int c, int nprob, double rel_tol,
                       double* sigma, int* order, int* kept, cplx* Qt, long long ldq, long long qstride,
                       void* ws, int* sweeps_out, cudaStream_t stream) {
  if (n <= 0 || c <= 0 || nprob <= 0 || ldw < n || ldq < n) return CIRR_EINVAL;
  unsigned char* base = reinterpret_cast<unsigned char*>(ws);
  unsigned* bar = reinterpret_cast<unsigned*>(base);
  int* counters = reinterpret_cast<int*>(base + 3072);  // after the barrier lines (<= 296 CTAs)
  cplx* Xc = reinterpret_cast<cplx*>(base + 4096);
  cplx* Jt = Xc + (long long)nprob * c * c;
  cplx* tau = Jt + (long long)nprob * c * c;
  cudaError_t e = cudaMemsetAsync(ws, 0, 4096, stream);
  if (e != cudaSuccess) return (int)e;
  // many small blocks: one CTA per problem, all in shared memory
  // (CIRR_ORTH_SMALL=0 forces the cooperative kernel)
  static const int small_env = getenv("CIRR_ORTH_SMALL") ? atoi(getenv("CIRR_ORTH_SMALL")) : 1;
  const long long osm = orth_small_smem(n, c);
  if (small_env != 0 && nprob >= 16 && n <= OS_NMAX && osm <= 200 * 1024) {
    if ((e = cudaMemsetAsync(sweeps_out, 0, sizeof(int), stream)) != cudaSuccess) return (int)e;
    cudaFuncSetAttribute(orth_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const double tol_s = 16.0 * sqrt((double)c) * 1.1102230246251565e-16;
    orth_small_kernel<<<nprob, OS_T, (size_t)osm, stream>>>(W, ldw, wstride, n, c, rel_tol, sigma, order, kept, Qt,
                                                            ldq, qstride, 60, tol_s, sweeps_out);
    CIRR_CHECK_LAUNCH();
    return 0;
  }
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int jb = JB_MAX;
  while (jb > 1 && sizeof(cplx) * 4 * jb * (size_t)c > 227 * 1024) jb >>= 1;
  const size_t jsmem = sizeof(cplx) * 4 * jb * (size_t)c;
  if (jsmem > 227 * 1024) return CIRR_EINVAL;
  cudaFuncSetAttribute(qr_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jsmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qr_jacobi_kernel, HT, jsmem);
  if (per_sm < 1) return CIRR_EINVAL;
  const int cp = c + (c & 1);
  long long want = (long long)nprob * (cp / 2);
  if (want < (long long)nprob * c) want = (long long)nprob * c;
  long long cap = (long long)sms * (per_sm < 2 ? per_sm : 2);
  if (g_cirr_coop_cap > 0 && cap > g_cirr_coop_cap) cap = g_cirr_coop_cap;
  int grid = (int)(want < cap ? want : cap);
  if (grid < 1) grid = 1;
  // rotation threshold on |x^H y| / (|x||y|) for length-c rows
  double tol = 16.0 * sqrt((double)c) * 1.1102230246251565e-16;
  int max_sweeps = 60;
  // C (Q = H_0 ... H_{c-1} [J_kept; 0]) as blocked WY products on the DMMA GEMM
  // for wide blocks; one reflector at a time inside the kernel for narrow ones
  static const int wy_env = getenv("CIRR_ORTH_WY") ? atoi(getenv("CIRR_ORTH_WY")) : -1;
  int back = (wy_env >= 0 ? wy_env == 0 : c < 64) ? 1 : 0;
  // A (Householder QR) blocked for wide blocks: panels of WYB columns plus WY
  // updates of the rest on the GEMM (CIRR_ORTH_QRB=0: one column at a time
  // inside the cooperative kernel)
  static const int qrb_env = getenv("CIRR_ORTH_QRB") ? atoi(getenv("CIRR_ORTH_QRB")) : -1;
  int do_qr = (qrb_env >= 0 ? qrb_env == 0 : (c < 64 || n < 1024)) ? 1 : 0;
  if (!do_qr) {
    int pcap = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pcap, qr_panel_kernel, HT, 0);
    pcap = sms * (pcap < 2 ? pcap : 2);
    if (g_cirr_coop_cap > 0 && pcap > g_cirr_coop_cap) pcap = g_cirr_coop_cap;
    CIRR_TRY(orth_qr_blocked(W, ldw, wstride, n, c, nprob, tau, bar, pcap < 1 ? 1 : pcap, stream));
  }
  void* args[] = {&W, &ldw, &wstride, &n, &c, &nprob, &rel_tol, &sigma, &order, &kept, &Qt, &ldq, &qstride,
                  &bar, &counters, &Xc, &Jt, &tau, &max_sweeps, &tol, &sweeps_out, &jb, &back, &do_qr};
  e = cudaLaunchCooperativeKernel((void*)qr_jacobi_kernel, dim3(grid), dim3(HT), args, jsmem, stream);
  cirr_note_launch();
  if (e != cudaSuccess) return (int)e;
  if (back) return 0;
  return orth_back_blocked(W, ldw, wstride, n, c, nprob, kept, order, Jt, tau, Qt, ldq, qstride, stream);
}

// --------------------------------------------------------------------------
// FEAST basis: Gram-Schmidt with re-orthogonalisation and column dropping.
//
// Replaces linalg.py:79-104 (orthonormalize: two MGS passes per column, drop a
// column whose norm falls below drop_tol * its original norm).  Classical
// Gram-Schmidt applied twice (CGS2) gives the same result to rounding and turns
// each pass into two parallel products; one CTA per problem, rows of length n
// (the columns of the block), fixed-order reductions.
namespace {
constexpr int GT2 = 512;
__global__ void __launch_bounds__(GT2) cgs2_kernel(const cplx* __restrict__ Y, long long ldy, long long sy, int n,
                                                   int c, double drop_tol, cplx* __restrict__ Qt, long long ldq,
                                                   long long sq, int* __restrict__ kept_out) {
  extern __shared__ cplx coef[];
  __shared__ double red[32];
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = GT2 / 32;
  const cplx* Yp = Y + (long long)p * sy;
  cplx* Q = Qt + (long long)p * sq;
  int kept = 0;
  for (int j = 0; j < c; ++j) {
    cplx* v = Q + (long long)kept * ldq;  // work in the next free output row
    double o2 = 0.0;
    for (int e = tid; e < n; e += GT2) {
      const cplx y = Yp[(long long)j * ldy + e];
      v[e] = y;
      o2 += cabs2(y);
    }
    const double orig = sqrt(block_sum(o2, red));
    if (orig == 0.0) continue;
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = wid; i < kept; i += nw) {
        const cplx* q = Q + (long long)i * ldq;
        double sr = 0.0, si = 0.0;
        for (int e = lane; e < n; e += 32) {
          const cplx g = cconjmul(q[e], v[e]);
          sr += g.x;
          si += g.y;
        }
        sr = warp_sum(sr);
        si = warp_sum(si);
        if (lane == 0) coef[i] = cmk(sr, si);
      }
      __syncthreads();
      for (int e = tid; e < n; e += GT2) {
        cplx x = v[e];
        for (int i = 0; i < kept; ++i) cfms(x, coef[i], Q[(long long)i * ldq + e]);
        v[e] = x;
      }
      __syncthreads();
    }
    double n2 = 0.0;
    for (int e = tid; e < n; e += GT2) n2 += cabs2(v[e]);
    const double nrm = sqrt(block_sum(n2, red));
    if (nrm <= drop_tol * orig) continue;
    const double inv = 1.0 / nrm;
    for (int e = tid; e < n; e += GT2) v[e] = cscale(v[e], inv);
    __syncthreads();
    ++kept;
  }
  if (tid == 0) kept_out[p] = kept;
}
}  // namespace

// Orthonormal basis of each block (rows of Y = columns of the block, c x n),
// dropping columns below drop_tol relative norm; Qt[p] rows 0..kept[p]-1.
CIRR_API int cirr_orthonormalize(const cplx* Y, long long ldy, long long sy, int n, int c, int nprob, double drop_tol,
                                 cplx* Qt, long long ldq, long long sq, int* kept, cudaStream_t stream) {
  if (n <= 0 || c <= 0 || nprob <= 0 || c > 4096) return CIRR_EINVAL;
  const size_t smem = sizeof(cplx) * (size_t)c;
  if (smem > 48 * 1024) cudaFuncSetAttribute(cgs2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cgs2_kernel<<<nprob, GT2, smem, stream>>>(Y, ldy, sy, n, c, drop_tol, Qt, ldq, sq, kept);
  CIRR_CHECK_LAUNCH();
  return 0;
}

// debug: clock64 marks of the last cirr_orth launch (start, after QR, after Jacobi, end)
CIRR_API int cirr_orth_phases(long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_orth_phase, sizeof(long long) * 4);
}

// --------------------------------------------------------------------------
// Certified CholeskyQR2: the fast basis for full-rank blocks.
//
// linalg.py:107-119 keeps the left singular vectors with sigma >= rel_tol *
// sigma_max.  When every sigma passes, that basis spans range(S), and the
// Rayleigh-Ritz values and vectors depend only on that span (up to rounding
// and the phase of each unit eigenvector).  So when S is certifiably full
// rank, an orthonormal basis from CholeskyQR2 (the north star's
// "CholeskyQR2 plus an SVD threshold") replaces the Householder QR + Jacobi
// SVD: Gram matrix on the DMMA GEMM, one-CTA Cholesky and triangular
// inverse, Q = S R^-1 on the GEMM, twice.  The certificate is
// kappa_F(R1) = ||R1||_F ||R1^-1||_F <= kappa_max (>= kappa_2(S), up to the
// rounding of the Gram matrix); with kappa_max far below both 1/rel_tol and
// eps^-1/2 the block is full rank and CholeskyQR2 is accurate.  Otherwise
// ok = 0 and the caller runs cirr_orth.
namespace {
constexpr int CT = 256;

// G (c x c, ld cmax) = S^H S  ->  R (upper, in place), RinvT = (R^-1)^T (cmax x cmax,
// zero outside c x c), ok &= certificate.  One CTA per problem.
__global__ void __launch_bounds__(CT) chol_inv_kernel(cplx* __restrict__ Gall, const int* __restrict__ cdim,
                                                      int cmax, double kappa_max, cplx* __restrict__ RinvT_all,
                                                      int* __restrict__ ok, int first_pass) {
  __shared__ double sred[32];
  __shared__ int s_fail;
  const int p = blockIdx.x, c = cdim[p], tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  cplx* G = Gall + (long long)p * cmax * cmax;
  cplx* RT = RinvT_all + (long long)p * cmax * cmax;
  for (int e = tid; e < cmax * cmax; e += CT) RT[e] = cmk(0.0, 0.0);
  if (tid == 0) s_fail = (c <= 0);
  __syncthreads();
  // right-looking Cholesky, upper factor in the upper triangle of G
  double dmax = 0.0;
  for (int j = 0; j < c; ++j) dmax = fmax(dmax, G[(long long)j * cmax + j].x);
  for (int j = 0; j < c && !s_fail; ++j) {
    const double d = G[(long long)j * cmax + j].x;
    if (!(d > 1e-300 && d > 1e-24 * dmax && d < 1e300)) {
      if (tid == 0) s_fail = 1;
      __syncthreads();
      break;
    }
    const double r = sqrt(d), ir = 1.0 / r;
    __syncthreads();
    if (tid == 0) G[(long long)j * cmax + j] = cmk(r, 0.0);
    for (int i = j + 1 + tid; i < c; i += CT) G[(long long)j * cmax + i] = cscale(G[(long long)j * cmax + i], ir);
    __syncthreads();
    const int rest = c - j - 1;
    for (int e = tid; e < rest * rest; e += CT) {
      const int a = j + 1 + e / rest, b = j + 1 + e % rest;
      if (b < a) continue;
      cfms(G[(long long)a * cmax + b], cconj(G[(long long)j * cmax + a]), G[(long long)j * cmax + b]);
    }
    __syncthreads();
  }
  __syncthreads();
  if (s_fail) {
    if (tid == 0) ok[p] = 0;
    return;
  }
  // R^-1 column by column (a warp per column, back substitution), stored transposed
  for (int j = wid; j < c; j += CT / 32) {
    for (int i = j; i >= 0; --i) {
      double sr = 0.0, si = 0.0;
      for (int k = i + 1 + lane; k <= j; k += 32) {
        const cplx g = cmul(G[(long long)i * cmax + k], RT[(long long)j * cmax + k]);
        sr += g.x;
        si += g.y;
      }
      sr = warp_sum(sr);
      si = warp_sum(si);
      if (lane == 0) {
        const cplx rhs = cmk((i == j ? 1.0 : 0.0) - sr, -si);
        RT[(long long)j * cmax + i] = cscale(rhs, 1.0 / G[(long long)i * cmax + i].x);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  // certificate on the first pass: ||R||_F ||R^-1||_F
  if (first_pass) {
    double a = 0.0, b = 0.0;
    for (int e = tid; e < c * c; e += CT) {
      const int i = e / c, k = e % c;
      if (k >= i) a += cabs2(G[(long long)i * cmax + k]);
      b += cabs2(RT[(long long)i * cmax + k]);
    }
    a = block_sum(a, sred);
    b = block_sum(b, sred);
    if (tid == 0) ok[p] = (sqrt(a) * sqrt(b) <= kappa_max) ? 1 : 0;
  }
}

// The same for c <= CSM_MAX with the factor in shared memory (packed upper
// triangle): Cholesky in place, then each thread back-substitutes one column
// of R^-1 (no inter-thread dependence, coalesced stores of R^-1 by rows into
// G), and a final transpose into RinvT.
constexpr int CSM_MAX = 160;
__device__ __forceinline__ int pk(int i, int k, int c) { return i * c - (i * (i - 1)) / 2 + (k - i); }

__global__ void __launch_bounds__(CT) chol_inv_smem_kernel(cplx* __restrict__ Gall, const int* __restrict__ cdim,
                                                           int cmax, double kappa_max, cplx* __restrict__ RinvT_all,
                                                           int* __restrict__ ok, int first_pass) {
  extern __shared__ __align__(16) cplx R[];
  __shared__ double sred[32];
  __shared__ int s_fail;
  const int p = blockIdx.x, c = cdim[p], tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = CT / 32;
  cplx* G = Gall + (long long)p * cmax * cmax;
  cplx* RT = RinvT_all + (long long)p * cmax * cmax;
  double dmax = 0.0;
  for (int i = 0; i < c; ++i) dmax = fmax(dmax, G[(long long)i * cmax + i].x);
  for (int e = tid; e < c * c; e += CT) {
    const int i = e / c, k = e % c;
    if (k >= i) R[pk(i, k, c)] = G[(long long)i * cmax + k];
  }
  for (int e = tid; e < cmax * cmax; e += CT) RT[e] = cmk(0.0, 0.0);
  if (tid == 0) s_fail = (c <= 0);
  __syncthreads();
  // Cholesky G = R^H R, packed upper rows in shared memory; the trailing
  // update maps a warp to a row and lanes to its columns (no index division)
  for (int j = 0; j < c; ++j) {
    const double d = R[pk(j, j, c)].x;
    if (!(d > 1e-300 && d > 1e-24 * dmax && d < 1e300)) {
      if (tid == 0) s_fail = 1;
      break;                                  // d is the same in every thread
    }
    const double r = sqrt(d), ir = 1.0 / r;
    __syncthreads();
    if (tid == 0) R[pk(j, j, c)] = cmk(r, 0.0);
    for (int i = j + 1 + tid; i < c; i += CT) R[pk(j, i, c)] = cscale(R[pk(j, i, c)], ir);
    __syncthreads();
    for (int a = j + 1 + wid; a < c; a += NW) {
      const cplx ca = cconj(R[pk(j, a, c)]);
      cplx* Ra = R + pk(a, a, c);          // row a from column a
      const cplx* Rj = R + pk(j, a, c);    // row j from column a
      for (int b = lane; b < c - a; b += 32) cfms(Ra[b], ca, Rj[b]);
    }
    __syncthreads();
  }
  __syncthreads();
  if (s_fail) {
    if (tid == 0) ok[p] = 0;
    return;
  }
  double a = 0.0;
  for (int e = tid; e < c * (c + 1) / 2; e += CT) a += cabs2(R[e]);
  if (first_pass) a = block_sum(a, sred);
  // X = R^-1 in place, column by column (R X = I, X upper):
  // X[0:j, j] = -X[0:j, 0:j] R[0:j, j] / R_jj, X_jj = 1 / R_jj; row i's dot
  // product in thread i.  The first version solved column j in thread j
  // reading R from global memory (one dependent L2 round trip per
  // multiply-add, ~1 ms per 118 x 118 factor on config 4's refinement rounds)
  for (int j = 0; j < c; ++j) {
    double sr0 = 0.0, si0 = 0.0, sr1 = 0.0, si1 = 0.0;
    const int i = tid;
    if (i < j) {
      const cplx* Xi = R + pk(i, i, c);     // X[i][k] = Xi[k - i]
      int k = i;
      for (; k + 1 < j; k += 2) {
        const cplx x0 = Xi[k - i], r0 = R[pk(k, j, c)];
        const cplx x1 = Xi[k + 1 - i], r1 = R[pk(k + 1, j, c)];
        sr0 = fma(x0.x, r0.x, sr0); sr0 = fma(-x0.y, r0.y, sr0);
        si0 = fma(x0.x, r0.y, si0); si0 = fma(x0.y, r0.x, si0);
        sr1 = fma(x1.x, r1.x, sr1); sr1 = fma(-x1.y, r1.y, sr1);
        si1 = fma(x1.x, r1.y, si1); si1 = fma(x1.y, r1.x, si1);
      }
      if (k < j) {
        const cplx x0 = Xi[k - i], r0 = R[pk(k, j, c)];
        sr0 = fma(x0.x, r0.x, sr0); sr0 = fma(-x0.y, r0.y, sr0);
        si0 = fma(x0.x, r0.y, si0); si0 = fma(x0.y, r0.x, si0);
      }
    }
    const double inv = 1.0 / R[pk(j, j, c)].x;
    __syncthreads();
    if (i < j) R[pk(i, j, c)] = cmk(-(sr0 + sr1) * inv, -(si0 + si1) * inv);
    if (i == j) R[pk(j, j, c)] = cmk(inv, 0.0);
    __syncthreads();
  }
  double b = 0.0;
  for (int e = tid; e < c * c; e += CT) {
    const int i = e / c, k = e % c;
    if (k >= i) {
      const cplx x = R[pk(i, k, c)];
      RT[(long long)k * cmax + i] = x;
      b += cabs2(x);
    }
  }
  if (first_pass) {
    b = block_sum(b, sred);
    if (tid == 0) ok[p] = (sqrt(a) * sqrt(b) <= kappa_max) ? 1 : 0;
  }
}
}  // namespace

CIRR_API long long cirr_orth_cholqr2_ws_bytes(int n, int c, int nprob) {
  return (long long)nprob * (2LL * n * c + 2LL * c * c) * 16 + 1024;
}

// W[p] (c x n rows: the columns of S) -> Qt[p] (cdim[p] orthonormal rows
// spanning the same space, zero rows after), ok[p] = certificate.  W is not
// modified.  ws: cirr_orth_cholqr2_ws_bytes.  No host synchronisation.
CIRR_API int cirr_orth_cholqr2(const cplx* W, long long ldw, long long wstride, int n, int c, int nprob,
                               const int* cdim, double kappa_max, cplx* Qt, long long ldq, long long qstride,
                               void* ws, int* ok, cudaStream_t stream) {
  if (n <= 0 || c <= 0 || nprob <= 0 || ldw < n || ldq < n || c > n) return CIRR_EINVAL;
  cplx* S = reinterpret_cast<cplx*>(ws);               // n x c per problem
  cplx* Q1 = S + (long long)nprob * n * c;             // c x n per problem
  cplx* G = Q1 + (long long)nprob * n * c;             // c x c
  cplx* RT = G + (long long)nprob * c * c;             // c x c
  const long long nc = (long long)n * c, cc = (long long)c * c;
  for (int pass = 0; pass < 2; ++pass) {
    const cplx* Wi = pass == 0 ? W : Q1;
    const long long ldi = pass == 0 ? ldw : n, si = pass == 0 ? wstride : nc;
    cplx* Wo = pass == 0 ? Q1 : Qt;
    const long long ldo = pass == 0 ? n : ldq, so = pass == 0 ? nc : qstride;
    CIRR_TRY(cirr_transpose(0, Wi, ldi, si, c, n, nprob, S, c, nc, stream));
    CIRR_TRY(cirr_gemm(1, c, c, n, nprob, Wi, ldi, si, S, c, nc, G, c, cc, 1.0, 0, stream));
    if (c <= CSM_MAX) {
      const int smem = (int)(sizeof(cplx) * ((long long)c * (c + 1) / 2));
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(chol_inv_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(cplx) * CSM_MAX * (CSM_MAX + 1) / 2));
        attr = true;
      }
      chol_inv_smem_kernel<<<nprob, CT, smem, stream>>>(G, cdim, c, kappa_max, RT, ok, pass == 0);
    } else {
      chol_inv_kernel<<<nprob, CT, 0, stream>>>(G, cdim, c, kappa_max, RT, ok, pass == 0);
    }
    CIRR_CHECK_LAUNCH();
    CIRR_TRY(cirr_gemm(0, c, n, c, nprob, RT, c, cc, Wi, ldi, si, Wo, ldo, so, 1.0, 0, stream));
  }
  return 0;
}
