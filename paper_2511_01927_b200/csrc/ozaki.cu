// Complex128 GEMM update C -= A B on the 5th-generation tensor cores by the
// Ozaki splitting: every row of A and every column of B is scaled by a power of
// two and cut into eight signed 7-bit digits (int8 slices; 6 + 7 x 7 = 55 bits
// below the row / column maximum), the digit products A_p B_q with p + q <= 7
// are exact int32 sums on tcgen05.mma kind::i8 (SASS UTCIMMA) accumulated in
// tensor memory per weight d = p + q (four accumulators of 128 columns fill
// the 512 TMEM columns, so a tile takes two passes: d = 0..3, then d = 4..7),
// and the epilogue recombines each pass's four accumulators in int64, converts
// once to FP64, applies the two scales and subtracts from C.  The truncation
// error per k-term is below 2^-53 rowmax(A) colmax(B): that of an FP64 GEMM up
// to the usual bound, with integer (order-independent, bitwise reproducible)
// accumulation.
//
// Replaces, for the k = 512 trailing updates of the dense LU and of the blocked
// solves, the DMMA kernel zgemm_sub_tma (lu_gemm.cuh): B200's FP64 tensor peak
// is 37.1 TF/s (measured, tools/fp64_peak.cu), its int8 tensor peak 4.57 POPS
// (measured, tools/i8_peak.cu); 36 slice products of the real 2m x 2n x 2k
// embedding cost 288 mnk int8 operations per 8 mnk flops.  Measured: 67 TF/s
// FP64-equivalent at the LU's largest update (DESIGN.md section 4,
// profiles/r02_ozaki_experiments.txt).
//
// Complex embedding: A' = [Re A | Im A] (m x 2k), and for complex column j of
// B two rows of B'^T: [Re b_j ; -Im b_j] (real part of the product) and
// [Im b_j ; Re b_j] (imaginary part), so the accumulator columns are
// interleaved (re, im) like complex128 memory.
//
// Execution: persistent CTA pairs (cta_group::2, M = 256 over the pair), TMA
// producer warp, one MMA-issuing thread in the pair's leader, eight epilogue
// warps per CTA; see the comments in ozaki_gemm_kernel.
//
// Reference: this is the arithmetic behind linalg.py:55-71 (splu of z_j B - A)
// and linalg.py:46-52 (its solves); the reference calls SuperLU in FP64.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cfloat>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "ozaki.cuh"

namespace cirr {
namespace {

constexpr int OS = 8;         // slices
constexpr int OBM = 128;      // accumulator rows = TMEM lanes
constexpr int OBN = 128;      // accumulator columns (real) = 64 complex columns
constexpr int OKB = 64;       // bytes of K' per stage (rows of the 64-byte swizzle) = two MMA K steps
constexpr int ONSTAGE = 3;
constexpr int OTHREADS = 320; // warp 0: TMA producer, warp 1: MMA issuer, warps 2-9: epilogue
constexpr int OBNH = OBN / 2;   // rows of a B slice tile held by each CTA of the pair (cta_group::2)
constexpr int OA_SLICE = OBM * OKB, OB_SLICE = OBNH * OKB;
constexpr int OSLOT_A = 4, OSLOT_B = 7;   // slice tiles a stage holds (largest sweep: 4 of A, 7 of B)
constexpr int OSTAGE = OSLOT_A * OA_SLICE + OSLOT_B * OB_SLICE;
constexpr int OSMEM = ONSTAGE * OSTAGE + 1024 + 256;

__device__ __forceinline__ unsigned osmem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ombar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(osmem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void ombar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}"
               ::"r"(osmem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ombar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(osmem_u32(bar)), "r"(parity) : "memory");
}
// wait with cluster-scope acquire (arrivals come from the other CTA of the pair)
__device__ __forceinline__ void ombar_wait_cluster(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAITC_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAITC_%=;\n}" ::"r"(osmem_u32(bar)), "r"(parity) : "memory");
}
// K-major operand tile with the 64-byte swizzle: rows of 64 bytes, groups of
// eight rows 512 bytes apart (stride byte offset), descriptor version 1,
// layout type 4 (SWIZZLE_64B).  A K step of 32 bytes advances the start address.
__device__ __forceinline__ uint64_t oumma_desc(unsigned saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * OKB) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(OKB == 64 ? 4 : 6) << 61;
  return d;
}
// TMA load into this CTA's shared memory, completion on the pair leader's barrier
__device__ __forceinline__ void otma_load4_pair(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                                unsigned leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(osmem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(leader_bar) : "memory");
}
__device__ __forceinline__ unsigned omapa(const void* p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(osmem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void ombar_arrive_cluster(unsigned cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void oumma2_i8(unsigned tmem_d, uint64_t da, uint64_t db, unsigned idesc, unsigned acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}"
      ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void oumma2_commit_mc(uint64_t* bar, unsigned short mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(osmem_u32(bar)), "h"(mask) : "memory");
}
__device__ __forceinline__ void ocluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned ocluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// 16 TMEM lanes x 32 columns: lane l of the warp gets, for repetition j = 0..3, columns
// 8 j + 2 (l % 4) + {0, 1} of row l / 4 (registers 4 j + 0, 1) and of row l / 4 + 8
// (registers 4 j + 2, 3): two adjacent accumulator columns = one complex element,
// four lanes = 64 contiguous bytes of a row of C.
__device__ __forceinline__ void otmem_ld_16x256b_x4(unsigned taddr, unsigned* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr) : "memory");
}

struct OzGeom {
  int M, N;          // rows, complex columns of C
  int K2;            // bytes of K' = 2 K
  int batch;
  int tiles_m, tiles_n;
  cplx* C; long long ldc, sC;
  const double* sa;  // [A tensor index][sa_stride]   2^(e_i - 6), row a_row0 + i
  const double* sb;  // [batch][N]   2^(f_j - 6)
  long long sa_stride;
  int a_row0;        // first row of A inside its slice tensor (TMA coordinate 1)
  int a_mul, a_add;  // A tensor index (TMA coordinate 3) of entry b: abatch(b) * a_mul + a_add
  const int* a_bmap; // optional: abatch(b) = a_bmap[b] (gathered solves), else b
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(OTHREADS, 1) ozaki_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                                                                 const __grid_constant__ CUtensorMap mapB, OzGeom g) {
  extern __shared__ __align__(1024) uint8_t osmem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)osmem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + ONSTAGE * OSTAGE);
  uint64_t* empty = full + ONSTAGE;
  uint64_t* tfull = empty + ONSTAGE;
  uint64_t* tempty = tfull + 1;
  unsigned* tmem_slot = (unsigned*)(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ONSTAGE; ++s) { ombar_init(&full[s], 1); ombar_init(&empty[s], 1); }
    ombar_init(tfull, 1);
    ombar_init(tempty, 16);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(osmem_u32(tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  ocluster_sync();   // both CTAs' barriers exist before any remote arrive or multicast
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = *tmem_slot;

  // A pair of CTAs (cta_group::2) takes two row tiles (2 tmp, 2 tmp + 1) of the
  // same column tile: each loads its own A slices and its half (64 rows) of the
  // B slices; the leader's MMAs (M = 256) make each tensor core read the other
  // half of B from the partner, so a CTA's shared-memory port carries 96 B/clk
  // of operand reads instead of 128.  Both CTAs run the same trip counts; the
  // leader's commits release the stages and publish the accumulators in both.
  const unsigned crank = ocluster_rank();
  const int tiles_mp = (g.tiles_m + 1) >> 1;
  const int per = tiles_mp * g.tiles_n;
  const int ntiles = per * g.batch;
  const int nkb = g.K2 / OKB;
  const int cl_id = blockIdx.x >> 1, cl_n = gridDim.x >> 1;

  // Every output tile (128 rows x 128 real columns) is produced in two passes:
  // pass 0 forms the accumulators of the weights d = 0..3 (one sweep over K:
  // 10 slice products among slices 0..3 of both operands), pass 1 those of
  // d = 4..7 in two sweeps over K (A 0..3 x B 1..7: 16 products, then A 4..7 x
  // B 0..3: 10 products), so a stage never holds more than 4 + 7 slice tiles
  // (88 KB; two stages).  Four 128-column accumulators fill the 512 TMEM
  // columns; with N = 128 an MMA reads (128 + 128) x 32 bytes of shared memory
  // per 64 tensor cycles -- exactly the 128 B/clk the SM delivers (N = 64 with
  // all eight accumulators side by side was bound there: 85 % shared-memory
  // pipe, 52 % tensor pipe, profiles/r02_ozaki_gemm_n64_raw.csv).
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = cl_id; t < ntiles; t += cl_n) {
        const int b = t / per, r = t - b * per;
        const int m0 = (2 * (r / g.tiles_n) + (int)crank) * OBM, n0 = (r % g.tiles_n) * OBN;
        // the last column tile is as narrow as the columns left (multiple of 16): each CTA holds half of it
        const int ntile = min(OBN, (2 * g.N - n0 + 15) & ~15);
        const int ab = (g.a_bmap ? g.a_bmap[b] : b) * g.a_mul + g.a_add;
        // sweep 0: A 0..3 x B 0..3 (d <= 3); sweep 1: A 0..3 x B 1..7 and sweep 2: A 4..7 x B 0..3 (d = 4..7)
        for (int sw = 0; sw < 3; ++sw) {
          const int a0 = sw == 2 ? 4 : 0, b0 = sw == 1 ? 1 : 0, nb = sw == 1 ? 7 : 4;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int st = it % ONSTAGE;
            const unsigned ph = (it / ONSTAGE) & 1;
            ombar_wait(&empty[st], ph ^ 1);
            // both CTAs' tiles complete on the leader's barrier (the MMA issuer lives there)
            if (crank == 0) ombar_arrive_expect_tx(&full[st], 2 * (4 * OA_SLICE + nb * OB_SLICE));
            const unsigned lbar = omapa(&full[st], 0);
            uint8_t* base = smem + st * OSTAGE;
            for (int s = 0; s < 4; ++s)
              otma_load4_pair(base + s * OA_SLICE, &mapA, kb * OKB, g.a_row0 + m0, a0 + s, ab, lbar);
            for (int s = 0; s < nb; ++s)
              otma_load4_pair(base + OSLOT_A * OA_SLICE + s * OB_SLICE, &mapB, kb * OKB, n0 + (int)crank * (ntile >> 1),
                              b0 + s, b, lbar);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {
      // instruction descriptor: D = S32, A = B = signed int8, both K-major, N >> 3, M >> 4 (M = 256 over the CTA pair)
      constexpr unsigned idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)((2 * OBM) >> 4) << 24);
      int it = 0, vt = 0;
      for (int t = cl_id; t < ntiles; t += cl_n) {
        const int n0 = ((t % per) % g.tiles_n) * OBN;
        const unsigned idesc = idesc0 | ((unsigned)(min(OBN, (2 * g.N - n0 + 15) & ~15) >> 3) << 17);
        for (int sw = 0; sw < 3; ++sw) {
          if (sw < 2) {  // sweeps 0 and 1 start a fresh accumulator set
            ombar_wait_cluster(tempty, (vt & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            ++vt;
          }
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int st = it % ONSTAGE;
            const unsigned ph = (it / ONSTAGE) & 1;
            ombar_wait(&full[st], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const unsigned abase = osmem_u32(smem + st * OSTAGE), bbase = abase + OSLOT_A * OA_SLICE;
#pragma unroll
            for (int ks = 0; ks < OKB / 32; ++ks) {
              const unsigned ak = abase + ks * 32, bk = bbase + ks * 32;
              if (sw == 0) {         // slots: A_p at p, B_q at q; d = p + q <= 3
#pragma unroll
                for (int d = 0; d < 4; ++d)
#pragma unroll
                  for (int p = 0; p <= d; ++p)
                    oumma2_i8(tmem + d * OBN, oumma_desc(ak + p * OA_SLICE), oumma_desc(bk + (d - p) * OB_SLICE),
                             idesc, (kb > 0 || ks > 0 || p > 0) ? 1u : 0u);
              } else if (sw == 1) {  // slots: A_p at p (p <= 3), B_q at q - 1 (q = 1..7); d = 4..7
#pragma unroll
                for (int d = 4; d < 8; ++d)
#pragma unroll
                  for (int p = 0; p < 4; ++p)
                    oumma2_i8(tmem + (d - 4) * OBN, oumma_desc(ak + p * OA_SLICE),
                             oumma_desc(bk + (d - p - 1) * OB_SLICE), idesc, (kb > 0 || ks > 0 || p > 0) ? 1u : 0u);
              } else {               // slots: A_p at p - 4 (p = 4..7), B_q at q (q <= 3); d = 4..7
#pragma unroll
                for (int d = 4; d < 8; ++d)
#pragma unroll
                  for (int p = 4; p <= d; ++p)
                    oumma2_i8(tmem + (d - 4) * OBN, oumma_desc(ak + (p - 4) * OA_SLICE),
                             oumma_desc(bk + (d - p) * OB_SLICE), idesc, 1u);
              }
            }
            oumma2_commit_mc(&empty[st], (unsigned short)3);
          }
          if (sw != 1) oumma2_commit_mc(tfull, (unsigned short)3);
        }
      }
    }
  } else {
    // Eight epilogue warps: warp w reads TMEM lanes 32 (w % 4) .. + 31 (its
    // hardware quadrant) and the 64-column half (w - 2) / 4 of the four
    // accumulators.  Their weighted sum is formed in one int64 and converted
    // once (weight 2^-21 after pass 0, 2^-49 after pass 1); the TMEM goes back
    // to the MMA warp before C is touched, so the next pass runs under this
    // pass's read-modify-write of C.  Both passes of an element are applied by
    // the same thread, in order.
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int tr = lane >> 2, tc = lane & 3;
    int vt = 0;
    for (int t = cl_id; t < ntiles; t += cl_n) {
      const int b = t / per, r = t - b * per;
      const int m0 = (2 * (r / g.tiles_n) + (int)crank) * OBM, n0 = (r % g.tiles_n) * OBN;
      // this thread: rows row0 + 16 hh + 8 rr (hh, rr in {0, 1}), complex columns col0 + 16 cg + 4 j (cg < 2, j < 4)
      const int row0 = m0 + quad * 32 + tr;
      const int col0 = (n0 >> 1) + half * 32 + tc;
      cplx* cbase = g.C + (long long)b * g.sC + (long long)row0 * g.ldc + col0;
      const double* sbp = g.sb + (long long)b * g.N + col0;
      const int ab = (g.a_bmap ? g.a_bmap[b] : b) * g.a_mul + g.a_add;
      const double* sap = g.sa + (long long)ab * g.sa_stride + g.a_row0 + row0;
      double sar[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rw = row0 + 8 * q;
        sar[q] = rw < g.M ? sap[8 * q] : 0.0;
        if (rw < g.M && col0 < g.N) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(cbase + (long long)(8 * q) * g.ldc));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(cbase + (long long)(8 * q) * g.ldc + 16));
        }
      }
      double sbc[8];
#pragma unroll
      for (int cj = 0; cj < 8; ++cj) sbc[cj] = (col0 + 4 * cj < g.N) ? sbp[4 * cj] : 0.0;
      for (int pass = 0; pass < 2; ++pass, ++vt) {
        const double pw = pass ? 0x1p-49 : 0x1p-21;
        double v[64];
        ombar_wait(tfull, vt & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int hc = 0; hc < 4; ++hc) {   // hc = 2 hh + cg
          unsigned v0[16], v1[16], v2[16], v3[16];
          const unsigned ta = tmem + ((unsigned)(quad * 32 + (hc >> 1) * 16) << 16) + half * 64 + (hc & 1) * 32;
          otmem_ld_16x256b_x4(ta + 0 * OBN, v0);
          otmem_ld_16x256b_x4(ta + 1 * OBN, v1);
          otmem_ld_16x256b_x4(ta + 2 * OBN, v2);
          otmem_ld_16x256b_x4(ta + 3 * OBN, v3);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j)
            v[hc * 16 + j] = (double)(((long long)(int)v0[j] << 21) + ((long long)(int)v1[j] << 14) +
                                      ((long long)(int)v2[j] << 7) + (long long)(int)v3[j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) ombar_arrive_cluster(omapa(tempty, 0));
        // C -= v sa sb: each warp instruction touches 8 rows x 64 contiguous bytes
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int q = 2 * hh + rr;
            if (row0 + 8 * q < g.M) {
              cplx* crow = cbase + (long long)(8 * q) * g.ldc;
              const double sr = sar[q] * pw;
              cplx cv[8];
#pragma unroll
              for (int cj = 0; cj < 8; ++cj)
                if (col0 + 4 * cj < g.N) cv[cj] = crow[4 * cj];
#pragma unroll
              for (int cj = 0; cj < 8; ++cj) {
                const int vi = (2 * hh + (cj >> 2)) * 16 + 4 * (cj & 3) + 2 * rr;
                const double sc = sr * sbc[cj];
                cv[cj].x = fma(-v[vi], sc, cv[cj].x);
                cv[cj].y = fma(-v[vi + 1], sc, cv[cj].y);
              }
#pragma unroll
              for (int cj = 0; cj < 8; ++cj)
                if (col0 + 4 * cj < g.N) crow[4 * cj] = cv[cj];
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  ocluster_sync();   // no multicast or remote arrive may land in a CTA that has left
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// Eight signed 7-bit digits of t (|t| < 64): t = sum_s d_s 2^(-7 s) up to 2^-49.
// Slice s of sixteen consecutive values packed into one 16-byte vector.
__device__ __forceinline__ void pack_slice(double (&t)[16], uint4& out, bool negate) {
  unsigned w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double d = rint(t[j]);
    t[j] = (t[j] - d) * 128.0;
    const int di = negate ? -(int)d : (int)d;
    w[j >> 2] |= ((unsigned)di & 0xffu) << (8 * (j & 3));
  }
  out = make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ uint4 negate_bytes(uint4 v) {
  // per-byte two's complement negation (digits lie in [-64, 64], no overflow)
  auto neg = [](unsigned x) { return __vsub4(0u, x); };
  return make_uint4(neg(v.x), neg(v.y), neg(v.z), neg(v.w));
}
__device__ __forceinline__ void scale_of(double mx, bool bad, double& scale, double& inv) {
  int e = 0;
  if (mx > 0.0) e = ilogb(mx) + 1;
  e = max(-1000, min(1024, e));   // 2^(e - 6) and 2^(6 - e) stay finite powers of two
  scale = bad ? nan("") : ldexp(1.0, e - 6);
  inv = ldexp(1.0, 6 - e);
}

// A (M x K complex, row-major) -> slices [batch][OS][M][2K] int8 and sa[batch][M].
// One warp per row.
__global__ void __launch_bounds__(256) ozaki_split_a_kernel(const cplx* __restrict__ A, long long lda, long long sA,
                                                            int M, int K, int8_t* __restrict__ out,
                                                            double* __restrict__ sa, int ob_mul, int ob_add) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp, b = blockIdx.y;
  if (row >= M) return;
  const cplx* a = A + (long long)b * sA + (long long)row * lda;
  double mx = 0.0;
  bool bad = false;
  for (int kk = lane; kk < K; kk += 32) {
    const cplx v = a[kk];
    const double m1 = fmax(fabs(v.x), fabs(v.y));
    bad |= !(fabs(v.x) <= DBL_MAX) || !(fabs(v.y) <= DBL_MAX);
    mx = fmax(mx, m1);
  }
  mx = warp_max(mx);
  bad = __any_sync(0xffffffffu, bad);
  double scale, inv;
  scale_of(mx, bad, scale, inv);
  const long long ob = (long long)b * ob_mul + ob_add;
  if (lane == 0) sa[ob * M + row] = scale;
  const long long K2 = 2LL * K;
  for (int kk0 = lane * 16; kk0 < K; kk0 += 512) {
    double tr[16], ti[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const cplx v = a[kk0 + j];
      tr[j] = bad ? 0.0 : v.x * inv;
      ti[j] = bad ? 0.0 : v.y * inv;
    }
#pragma unroll
    for (int s = 0; s < OS; ++s) {
      uint4 pr, pi;
      pack_slice(tr, pr, false);
      pack_slice(ti, pi, false);
      int8_t* o = out + ((ob * OS + s) * M + row) * K2;
      *reinterpret_cast<uint4*>(o + kk0) = pr;
      *reinterpret_cast<uint4*>(o + K + kk0) = pi;
    }
  }
}

// Column maxima of B (K x N complex, row-major): sb[batch][N].
__global__ void __launch_bounds__(256) ozaki_colscale_kernel(const cplx* __restrict__ B, long long ldb, long long sB,
                                                             int K, int N, double* __restrict__ sb) {
  const int j = blockIdx.x * 256 + threadIdx.x, b = blockIdx.y;
  if (j >= N) return;
  const cplx* p = B + (long long)b * sB + j;
  double mx = 0.0;
  bool bad = false;
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    const cplx v = p[(long long)k * ldb];
    const double m1 = fmax(fabs(v.x), fabs(v.y));
    bad |= !(fabs(v.x) <= DBL_MAX) || !(fabs(v.y) <= DBL_MAX);
    mx = fmax(mx, m1);
  }
  double scale, inv;
  scale_of(mx, bad, scale, inv);
  sb[(long long)b * N + j] = scale;
}

// B (K x N complex, row-major) -> slices [batch][OS][2N][2K] int8 (row 2j:
// [Re b_j ; -Im b_j], row 2j+1: [Im b_j ; Re b_j]).  A thread takes column j
// and sixteen consecutive k.
__global__ void __launch_bounds__(256) ozaki_split_b_kernel(const cplx* __restrict__ B, long long ldb, long long sB,
                                                            int K, int N, const double* __restrict__ sb,
                                                            int8_t* __restrict__ out) {
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int kk0 = (blockIdx.y * 8 + (threadIdx.x >> 5)) * 16;
  const int b = blockIdx.z;
  if (j >= N || kk0 >= K) return;
  const double scale = sb[(long long)b * N + j];
  const bool bad = !(scale <= DBL_MAX);
  const double inv = bad ? 0.0 : 1.0 / scale;
  const cplx* p = B + (long long)b * sB + (long long)kk0 * ldb + j;
  double tr[16], ti[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const cplx v = p[(long long)t * ldb];
    tr[t] = bad ? 0.0 : v.x * inv;
    ti[t] = bad ? 0.0 : v.y * inv;
  }
  const long long K2 = 2LL * K;
#pragma unroll
  for (int s = 0; s < OS; ++s) {
    uint4 pr, pi;
    pack_slice(tr, pr, false);
    pack_slice(ti, pi, false);
    int8_t* o = out + (((long long)b * OS + s) * (2LL * N) + 2 * j) * K2;
    *reinterpret_cast<uint4*>(o + kk0) = pr;
    *reinterpret_cast<uint4*>(o + K + kk0) = negate_bytes(pi);
    *reinterpret_cast<uint4*>(o + K2 + kk0) = pi;
    *reinterpret_cast<uint4*>(o + K2 + K + kk0) = pr;
  }
}

// B (K x N complex, row-major, K <= 512) -> column scales and slices in one
// launch: a CTA takes eight columns of one entry, stages the K x 8 block in
// shared memory (128-byte rows of B: coalesced), reduces the column maxima,
// and for every slice writes the sixteen rows (2j: [Re b_j ; -Im b_j], 2j+1:
// [Im b_j ; Re b_j]) -- contiguous in the slice tensor -- through a 16 KB
// staging block as one coalesced copy.  Replaces ozaki_colscale_kernel +
// ozaki_split_b_kernel (thread-per-column maxima, scattered 16-byte stores).
constexpr int OFB_COLS = 8, OFB_KMAX = 512, OFB_KP = OFB_KMAX + 4;
constexpr int OFB_SMEM = 2 * OFB_COLS * OFB_KP * 8 + 2 * OFB_COLS * 2 * OFB_KMAX + 1024;
__global__ void __launch_bounds__(256) ozaki_split_b_fused_kernel(const cplx* __restrict__ B, long long ldb,
                                                                  long long sB, int K, int N, double* __restrict__ sb,
                                                                  int8_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t fsm[];
  double* pre = reinterpret_cast<double*>(fsm);                 // [8][KP]
  double* pim = pre + OFB_COLS * OFB_KP;                        // [8][KP]
  int8_t* stage = reinterpret_cast<int8_t*>(pim + OFB_COLS * OFB_KP);   // [16 rows][2K]
  double* cmax = reinterpret_cast<double*>(stage + 2 * OFB_COLS * 2 * OFB_KMAX);  // [8 warps][8] then [8]
  __shared__ int sbad[OFB_COLS];
  const int j0 = blockIdx.x * OFB_COLS, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncol = min(OFB_COLS, N - j0);
  if (threadIdx.x < OFB_COLS) sbad[threadIdx.x] = 0;
  __syncthreads();
  {  // load: thread (k = t / 8 + 32 i, c = t % 8); a warp reads four 128-byte rows
    const int c = threadIdx.x & 7;
    const cplx* p = B + (long long)b * sB + j0 + c;
    double mx = 0.0;
    bool bad = false;
    for (int k = threadIdx.x >> 3; k < K; k += 32) {
      cplx v = cmk(0.0, 0.0);
      if (c < ncol) v = p[(long long)k * ldb];
      pre[c * OFB_KP + k] = v.x;
      pim[c * OFB_KP + k] = v.y;
      bad |= !(fabs(v.x) <= DBL_MAX) || !(fabs(v.y) <= DBL_MAX);
      mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
    }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    if (lane < 8) cmax[warp * 8 + lane] = mx;
    if (bad) sbad[c] = 1;
  }
  __syncthreads();
  if (threadIdx.x < OFB_COLS) {
    double mx = 0.0;
    for (int w = 0; w < 8; ++w) mx = fmax(mx, cmax[w * 8 + threadIdx.x]);
    double scale, inv;
    scale_of(mx, sbad[threadIdx.x] != 0, scale, inv);
    if ((int)threadIdx.x < ncol) sb[(long long)b * N + j0 + threadIdx.x] = scale;
    cmax[64 + threadIdx.x] = sbad[threadIdx.x] ? 0.0 : inv;
  }
  __syncthreads();
  // digits: warp = column, lane = k mod 32 (conflict-free reads of the planes)
  const int c = warp;
  const double inv = cmax[64 + c];
  double tr[16], ti[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int k = lane + 32 * i;
    tr[i] = k < K ? pre[c * OFB_KP + k] * inv : 0.0;
    ti[i] = k < K ? pim[c * OFB_KP + k] * inv : 0.0;
  }
  const int K2 = 2 * K;
  const long long rows2n = 2LL * N;
  // each warp stages and writes its own two rows (2 K2 contiguous bytes of the slice tensor): no CTA barrier
  int8_t* r0 = stage + (2 * c) * K2;       // row 2j:   [re ; -im]
  int8_t* r1 = r0 + K2;                    // row 2j+1: [im ;  re]
  const bool live = c < ncol;
  for (int s = 0; s < OS; ++s) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = lane + 32 * i;
      const double dr = rint(tr[i]), di = rint(ti[i]);
      tr[i] = (tr[i] - dr) * 128.0;
      ti[i] = (ti[i] - di) * 128.0;
      if (k < K) {
        const int8_t br = (int8_t)(int)dr, bi = (int8_t)(int)di;
        r0[k] = br;
        r0[K + k] = (int8_t)(-(int)di);
        r1[k] = bi;
        r1[K + k] = br;
      }
    }
    __syncwarp();
    if (live) {
      int8_t* dst = out + (((long long)b * OS + s) * rows2n + 2LL * (j0 + c)) * K2;
      const int nvec = (2 * K2) >> 4;
      for (int v = lane; v < nvec; v += 32)
        reinterpret_cast<uint4*>(dst)[v] = reinterpret_cast<const uint4*>(r0)[v];
    }
    __syncwarp();
  }
}

// column scales + slices of B: the fused kernel for K <= 512, else the two-kernel path
int split_b(const cplx* B, long long ldb, long long sB, int K, int N, int batch, double* sb, int8_t* wb,
            cudaStream_t stream) {
  if (K <= OFB_KMAX) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(ozaki_split_b_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OFB_SMEM);
      attr = true;
    }
    ozaki_split_b_fused_kernel<<<dim3((N + OFB_COLS - 1) / OFB_COLS, batch), 256, OFB_SMEM, stream>>>(B, ldb, sB, K, N,
                                                                                                     sb, wb);
    cirr_note_launch();
    return 0;
  }
  ozaki_colscale_kernel<<<dim3((N + 255) / 256, batch), 256, 0, stream>>>(B, ldb, sB, K, N, sb);
  cirr_note_launch();
  ozaki_split_b_kernel<<<dim3((N + 31) / 32, (K + 127) / 128, batch), 256, 0, stream>>>(B, ldb, sB, K, N, sb, wb);
  cirr_note_launch();
  return 0;
}

int encode_slice_map(CUtensorMap* map, const int8_t* base, long long K2, long long rows, long long batch,
                     int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return (int)cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[4] = {(cuuint64_t)K2, (cuuint64_t)rows, (cuuint64_t)OS, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)K2, (cuuint64_t)(K2 * rows), (cuuint64_t)(K2 * rows * OS)};
  cuuint32_t box[4] = {(cuuint32_t)OKB, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, OKB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}


// ---- factor slices kept for the solves ------------------------------------
// The factors do not change between the solve passes of a CIRR run, so their
// slices are cut once after the factorisation (cirr_ozaki_split_factors) into a
// caller-owned buffer and every k = 512 trailing update of the blocked solves
// reads them: per factor and 512-column block sb a tensor [OS][n][1024] of the
// rows' digits over those columns (rows above the block are U's, rows below
// L's), plus the row scales [n].
struct OzCache {
  const cplx* LU;
  long long pstride;
  int n, nfac, nsb;
  int8_t* slices;
  double* scales;
};
constexpr int OZ_W = 512;
constexpr int OZ_MAXCACHE = 16;
OzCache g_oz_cache[OZ_MAXCACHE];
int g_oz_ncache = 0;
std::mutex g_oz_mutex;

bool oz_lookup(const cplx* LU, int n, OzCache& out, long long& f0) {
  std::lock_guard<std::mutex> lk(g_oz_mutex);
  for (int i = 0; i < g_oz_ncache; ++i) {
    const OzCache& c = g_oz_cache[i];
    if (c.n != n || LU < c.LU) continue;
    const long long d = LU - c.LU;
    if (d % c.pstride != 0 || d / c.pstride >= c.nfac) continue;
    out = c;
    f0 = d / c.pstride;
    return true;
  }
  return false;
}


// Slice workspace: one buffer per launching stream, kept between calls and
// grown on demand (cudaMalloc; stream-ordered reuse is safe because every user
// of a stream's buffer runs on that stream).  cudaMallocAsync is not used here:
// a multi-GiB request blocked the host for 40-600 ms per call once PyTorch's
// allocator held most of the device (tools/gap_probe.py).
struct OzWs { cudaStream_t stream; void* p; size_t bytes; };
OzWs g_oz_ws[16];
int g_oz_nws = 0;

void* oz_workspace(cudaStream_t stream, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_oz_mutex);
  OzWs* w = nullptr;
  for (int i = 0; i < g_oz_nws; ++i)
    if (g_oz_ws[i].stream == stream) w = &g_oz_ws[i];
  if (!w) {
    if (g_oz_nws == 16) {   // a 17th stream: the oldest buffer goes (cudaFree synchronises the device)
      if (g_oz_ws[0].p) cudaFree(g_oz_ws[0].p);
      for (int i = 1; i < 16; ++i) g_oz_ws[i - 1] = g_oz_ws[i];
      --g_oz_nws;
    }
    w = &g_oz_ws[g_oz_nws++];
    *w = OzWs{stream, nullptr, 0};
  }
  if (w->bytes < bytes) {
    if (w->p) cudaFree(w->p);   // synchronises: no kernel still reads the old buffer
    w->p = nullptr;
    w->bytes = 0;
    const size_t want = (bytes + (64u << 20) - 1) & ~(size_t)((64u << 20) - 1);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {   // PyTorch's cache may hold the memory: the stream-ordered allocator's handler frees it
      cudaGetLastError();
      void* probe = nullptr;
      if (cirr_malloc_async(&probe, want, stream) == cudaSuccess) {
        cudaFreeAsync(probe, stream);
        cudaStreamSynchronize(stream);
        e = cudaMalloc(&p, want);
      }
      if (e != cudaSuccess) { cudaGetLastError(); return nullptr; }
    }
    w->p = p;
    w->bytes = want;
  }
  return w->p;
}

}  // namespace

long long ozaki_factor_bytes(int n, int nfac) {
  if (n < 2 * OZ_W || n % OZ_W != 0 || nfac <= 0) return 0;
  const long long nsb = n / OZ_W;
  return (long long)nfac * nsb * ((long long)OS * n * 2 * OZ_W + 8LL * n) + 512;
}

int ozaki_split_factors(const cplx* LU, int n, long long ld, long long pstride, int nfac, void* cache,
                        cudaStream_t stream) {
  if (ozaki_factor_bytes(n, nfac) == 0 || cache == nullptr) return CIRR_EINVAL;
  const int nsb = n / OZ_W;
  OzCache c{LU, pstride, n, nfac, nsb, reinterpret_cast<int8_t*>(cache), nullptr};
  const long long slice_bytes = (long long)nfac * nsb * OS * n * 2 * OZ_W;
  c.scales = reinterpret_cast<double*>(c.slices + ((slice_bytes + 255) & ~255LL));
  for (int sb = 0; sb < nsb; ++sb) {
    ozaki_split_a_kernel<<<dim3((n + 7) / 8, nfac), 256, 0, stream>>>(LU + (long long)sb * OZ_W, ld, pstride, n, OZ_W,
                                                                       c.slices, c.scales, nsb, sb);
    CIRR_CHECK_LAUNCH();
  }
  std::lock_guard<std::mutex> lk(g_oz_mutex);
  for (int i = 0; i < g_oz_ncache; ++i)
    if (g_oz_cache[i].LU == LU) { g_oz_cache[i] = c; return 0; }
  if (g_oz_ncache == OZ_MAXCACHE) {  // oldest entry out
    for (int i = 1; i < OZ_MAXCACHE; ++i) g_oz_cache[i - 1] = g_oz_cache[i];
    --g_oz_ncache;
  }
  g_oz_cache[g_oz_ncache++] = c;
  return 0;
}

// Drop every registration whose factors overlap [p, p + bytes): called by the
// LU itself (new factors in that memory make the slices stale) and by release.
void ozaki_invalidate(const void* p, long long bytes) {
  std::lock_guard<std::mutex> lk(g_oz_mutex);
  const char* lo = reinterpret_cast<const char*>(p);
  const char* hi = lo + bytes;
  int k = 0;
  for (int i = 0; i < g_oz_ncache; ++i) {
    const OzCache& c = g_oz_cache[i];
    const char* clo = reinterpret_cast<const char*>(c.LU);
    const char* chi = clo + ((long long)(c.nfac - 1) * c.pstride + (long long)c.n * c.n) * 16;
    if (clo < hi && lo < chi) continue;
    g_oz_cache[k++] = c;
  }
  g_oz_ncache = k;
}

int ozaki_release(const cplx* LU) {
  ozaki_invalidate(LU, 16);
  return 0;
}

// C -= A B where A = rows a_row0 .. a_row0 + M of the factor's column block
// col0 .. col0 + 512, read from the slices kept by ozaki_split_factors; entry b
// uses factor (LU - registered base) / stride + (pmap ? pmap[b] : b).  Returns
// -1 when the slices are not there (the caller takes the DMMA path).
int ozaki_cached_update(const cplx* LU, int n, int col0, int kw, int a_row0, int M, const cplx* B, long long ldb,
                        long long sB, cplx* C, long long ldc, long long sC, int N, int batch, const int* pmap,
                        cudaStream_t stream) {
  if (!ozaki_enabled() || kw != OZ_W || col0 % OZ_W != 0 || M <= 0 || N <= 0 || batch <= 0) return -1;
  OzCache c;
  long long f0 = 0;
  if (!oz_lookup(LU, n, c, f0)) return -1;
  const long long K2 = 2LL * OZ_W;
  const long long b_bytes = (long long)OS * 2 * N * K2;
  const size_t wb_bytes = ((size_t)batch * b_bytes + 255) & ~(size_t)255;
  int8_t* wb = reinterpret_cast<int8_t*>(oz_workspace(stream, wb_bytes + (size_t)batch * N * sizeof(double)));
  if (!wb) return (int)cudaErrorMemoryAllocation;
  double* sb = reinterpret_cast<double*>(wb + wb_bytes);
  int rc = 0;
  split_b(B, ldb, sB, OZ_W, N, batch, sb, wb, stream);
  CUtensorMap mA, mB;
  if (encode_slice_map(&mA, c.slices, K2, n, (long long)c.nfac * c.nsb, OBM) != 0 ||
      encode_slice_map(&mB, wb, K2, 2LL * N, batch, OBNH) != 0) {
    rc = (int)cudaErrorInvalidValue;
  } else {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaFuncSetAttribute(ozaki_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OSMEM);
    }
    OzGeom g{};
    g.M = M; g.N = N; g.K2 = (int)K2; g.batch = batch;
    g.tiles_m = (M + OBM - 1) / OBM;
    g.tiles_n = (2 * N + OBN - 1) / OBN;
    g.C = C; g.ldc = ldc; g.sC = sC;
    g.sa = c.scales; g.sb = sb;
    g.sa_stride = n; g.a_row0 = a_row0;
    g.a_mul = c.nsb; g.a_add = (int)(f0 * c.nsb + col0 / OZ_W);
    g.a_bmap = pmap;
    const long long npairs = (long long)((g.tiles_m + 1) / 2) * g.tiles_n * batch;
    ozaki_gemm_kernel<<<2 * (int)min((long long)(sms / 2), npairs), OTHREADS, OSMEM, stream>>>(mA, mB, g);
    cirr_note_launch();
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) rc = (int)le;
  }
  return rc;
}

namespace {
}  // namespace

// 0: FP64 DMMA trailing updates; 1 (default): int8 tensor-core (Ozaki) trailing
// updates for the dense LU's k = 512 steps and the blocked solves.
// CIRR_LU_GEMM=dmma | int8 sets the initial mode, cirr_set_lu_gemm changes it.
int g_cirr_lu_gemm = [] {
  const char* e = getenv("CIRR_LU_GEMM");
  if (!e) return 1;
  return (e[0] == 'd' || e[0] == 'f' || e[0] == '0') ? 0 : 1;
}();

bool ozaki_enabled() { return g_cirr_lu_gemm == 1; }

bool ozaki_shape_ok(int M, int N, int K) { return M > 0 && N > 0 && K >= 32 && K % 32 == 0 && K <= 4096; }

long long ozaki_ws_bytes_per_entry(int M, int N, int K) {
  return (long long)OS * 2 * K * ((long long)M + 2LL * N) + 8LL * (M + N) + 512;
}

// C -= A B for `batch` independent complex128 problems (row-major; strides in
// elements).  The slices of a chunk of entries (CIRR_OZAKI_WS_MB, default
// 512 MiB) live in the stream's kept workspace (oz_workspace).
int ozaki_zgemm_sub(const cplx* A, long long lda, long long sA, const cplx* B, long long ldb, long long sB, cplx* C,
                    long long ldc, long long sC, int M, int N, int K, int batch, cudaStream_t stream) {
  if (!ozaki_shape_ok(M, N, K) || batch <= 0) return CIRR_EINVAL;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ozaki_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OSMEM);
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  static const long long ws_mb = getenv("CIRR_OZAKI_WS_MB") ? atoll(getenv("CIRR_OZAKI_WS_MB")) : 512;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const long long K2 = 2LL * K;
  const long long a_bytes = (long long)OS * M * K2, b_bytes = (long long)OS * 2 * N * K2;
  const long long per = a_bytes + b_bytes;
  int chunk = (int)max(1LL, min((long long)batch, (ws_mb << 20) / per));
  const size_t slice_bytes = ((size_t)chunk * per + 255) & ~(size_t)255;
  int8_t* ws = reinterpret_cast<int8_t*>(oz_workspace(stream, slice_bytes + (size_t)chunk * (M + N) * sizeof(double)));
  if (!ws) return (int)cudaErrorMemoryAllocation;
  double* scales = reinterpret_cast<double*>(ws + slice_bytes);
  int rc = 0;
  for (int b0 = 0; b0 < batch && rc == 0; b0 += chunk) {
    const int nb = min(chunk, batch - b0);
    int8_t* wa = ws;
    int8_t* wb = ws + (long long)nb * a_bytes;
    double* sa = scales;
    double* sb = scales + (long long)nb * M;
    ozaki_split_a_kernel<<<dim3((M + 7) / 8, nb), 256, 0, stream>>>(A + (long long)b0 * sA, lda, sA, M, K, wa, sa, 1, 0);
    cirr_note_launch();
    split_b(B + (long long)b0 * sB, ldb, sB, K, N, nb, sb, wb, stream);
    CUtensorMap mA, mB;
    if (encode_slice_map(&mA, wa, K2, M, nb, OBM) != 0 || encode_slice_map(&mB, wb, K2, 2LL * N, nb, OBNH) != 0) {
      rc = (int)cudaErrorInvalidValue;
      break;
    }
    OzGeom g{};
    g.M = M; g.N = N; g.K2 = (int)K2; g.batch = nb;
    g.tiles_m = (M + OBM - 1) / OBM;
    g.tiles_n = (2 * N + OBN - 1) / OBN;
    g.C = C + (long long)b0 * sC; g.ldc = ldc; g.sC = sC;
    g.sa = sa; g.sb = sb;
    g.sa_stride = M; g.a_row0 = 0; g.a_mul = 1; g.a_add = 0; g.a_bmap = nullptr;
    const long long npairs = (long long)((g.tiles_m + 1) / 2) * g.tiles_n * nb;
    const int grid = 2 * (int)min((long long)(sms / 2), npairs);
    ozaki_gemm_kernel<<<grid, OTHREADS, OSMEM, stream>>>(mA, mB, g);
    cirr_note_launch();
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) rc = (int)le;
  }
  return rc;
}

}  // namespace cirr

CIRR_API long long cirr_ozaki_factor_bytes(int n, int nfac) { return cirr::ozaki_factor_bytes(n, nfac); }
CIRR_API int cirr_ozaki_split_factors(const cirr_cplx* LU, int n, long long ld, long long pencil_stride, int nfac,
                                      void* cache, cudaStream_t stream) {
  return cirr::ozaki_split_factors(LU, n, ld, pencil_stride, nfac, cache, stream);
}
CIRR_API int cirr_ozaki_release(const cirr_cplx* LU) { return cirr::ozaki_release(LU); }

CIRR_API int cirr_set_lu_gemm(int mode) {
  const int prev = cirr::g_cirr_lu_gemm;
  if (mode == 0 || mode == 1) cirr::g_cirr_lu_gemm = mode;
  return prev;
}

// C-ABI entry: C -= A B through the Ozaki int8 path (tests/test_gpu_ozaki.py).
CIRR_API int cirr_ozaki_zgemm_sub(const cirr_cplx* A, long long lda, long long sA, const cirr_cplx* B, long long ldb,
                                  long long sB, cirr_cplx* C, long long ldc, long long sC, int M, int N, int K,
                                  int batch, cudaStream_t stream) {
  return cirr::ozaki_zgemm_sub(A, lda, sA, B, ldb, sB, C, ldc, sC, M, N, K, batch, stream);
}
