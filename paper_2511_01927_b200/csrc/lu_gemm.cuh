// Persistent, warp-specialised complex128 GEMM  C[b] -= A[b] @ B[b]  for the
// LU trailing update (A22 -= L21 U12), with every operand tile moved by the
// Tensor Memory Accelerator.
//
// One CTA per SM loops over 64x64 output tiles of all pencils.  A producer
// warp issues one cp.async.bulk.tensor (TMA, SASS UTMALDG) per operand tile
// -- a 64x16 slice of L21, a 16x64 slice of U12 and the 64x64 C block -- into
// a 4-stage ring (completion by mbarrier transaction bytes; the L21 slice is
// two 64x8 boxes with the 128-byte swizzle so the DMMA A-fragment loads are
// bank-conflict free); out-of-range rows
// and columns are zero-filled by the TMA unit.  The C block of a tile is
// requested while that tile's main loop runs and the next tile's K slices
// during its epilogue, so HBM traffic for C overlaps tensor work.  Eight
// consumer warps run the complex DMMA main loop (mma.sync m8n8k4 f64 -> SASS
// DMMA.8x8x4) with two accumulator sets (re, im) per 8x8 block and write
// C - acc straight to global memory.
//
// The three tensor maps describe the whole pencil batch as a 3-D float64
// tensor {2n, n, batch} (complex128 = two doubles), so one encoding serves
// every panel step of a factorisation.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"

namespace cirr {

constexpr int PBM = 64, PBN = 64, PBK = 16, PSTAGES = 4;
constexpr int PCONS = 8;         // consumer warps
constexpr int PTHREADS = (PCONS + 1) * 32;
constexpr int P_A_BYTES = PBM * PBK * 16;
constexpr int PRING = 8;                        // tile-id ring (producer runs <= PSTAGES tiles ahead)
constexpr int PAK = 8;                          // complex columns per swizzled A box (128 bytes)
constexpr int P_A_HALF = PBM * PAK * 16;        // one A box
constexpr int P_B_BOX = PBK * PAK * 16;         // one swizzled 16 x 8 B box (2 KB)

// Output tiles are 64 x BN.  The LU uses BN = 64; the blocked solves pick BN
// from {64, 56, 48, 40, 32} to fit the right-hand-side width K (pick_tile_n:
// the first pass's K = 32 runs as one 32-wide tile instead of a half-empty
// 64-wide one).  Each consumer warp owns WI
// 8-row blocks x WJ 8-column blocks of the tile (8 warps cover 8 x BN/8 blocks).
//
// BSW (the solves): the B slice arrives as BN/8 boxes of 16 x 8 with the
// 128-byte swizzle, and the four k of each DMMA step are k = 2q + s inside an
// 8-wide box (q = lane % 4, s = step parity), so the A- and B-fragment loads
// of every quarter-warp hit eight distinct 16-byte bank groups.  Unswizzled,
// the B loads are 4-way conflicted: harmless at BN = 64 (6 loads per 32 DMMAs;
// the LU keeps it, the extra boxes cost it 0.6 %), but the narrow tiles (one
// A and up to seven B loads per 4 WJ DMMAs) were shared-memory bound.
template <int BN>
struct TileCfg;
template <> struct TileCfg<64> { static constexpr int WI = 4, WJ = 2; };
template <> struct TileCfg<56> { static constexpr int WI = 1, WJ = 7; };
template <> struct TileCfg<48> { static constexpr int WI = 2, WJ = 3; };
template <> struct TileCfg<40> { static constexpr int WI = 1, WJ = 5; };
template <> struct TileCfg<32> { static constexpr int WI = 2, WJ = 2; };
template <int BN>
struct TileBytes {
  static constexpr int B = PBK * BN * 16;
  static constexpr int STAGE = P_A_BYTES + B;
  static constexpr int C = PBM * BN * 16;
  static constexpr int SMEM = PSTAGES * STAGE + C + 8 * (2 * PSTAGES + 2) + 4 * PRING + 1024;
};
constexpr int P_STAGE_BYTES = TileBytes<64>::STAGE;
constexpr int P_C_BYTES = TileBytes<64>::C;
constexpr int P_SMEM = TileBytes<64>::SMEM;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ cplx lds_c(unsigned addr) {
  cplx v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}
// TMA tile load of a 3-D box at (c0, c1, c2) (c0 in doubles), completion on `bar`
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

struct SubGemmGeom {
  int M, N, K, batch;
  int a_row0, a_col0;   // L21 origin (rows, complex columns) inside each pencil
  int b_row0, b_col0;   // U12 origin
  int c_row0, c_col0;   // A22 origin
  cplx* C; long long ldc, sC;
  int tiles_m, tiles_n;
  int beta;        // 1: C = C - A B (C tile streamed in by TMA); 0: C = A B
  int a_bmul, a_badd;  // 3rd TMA coordinate of the A operand: b * a_bmul + a_badd
  int* ctr;            // {next tile, finished CTAs}: dynamic tile scheduler, zero on entry and exit
  const int* a_bmap;   // optional: the A operand of batch entry b is A entry a_bmap[b] (gathered solves)
};

template <int BN, bool BSW>
static __global__ void __launch_bounds__(PTHREADS, 1) zgemm_sub_tma(const __grid_constant__ CUtensorMap mapA,
                                                             const __grid_constant__ CUtensorMap mapB,
                                                             const __grid_constant__ CUtensorMap mapC,
                                                             SubGemmGeom g) {
  constexpr int WI = TileCfg<BN>::WI, WJ = TileCfg<BN>::WJ;
  constexpr int WARPS_N = (BN / 8) / WJ;
  static_assert((8 / WI) * WARPS_N == PCONS, "warp layout must cover the tile");
  constexpr int STAGE = TileBytes<BN>::STAGE, CBYTES = TileBytes<BN>::C;
  extern __shared__ __align__(1024) unsigned char psm_raw[];
  // 1024-byte alignment for the swizzled A boxes, kept in the shared window
  unsigned char* psm = psm_raw + ((1024u - (smem_u32(psm_raw) & 1023u)) & 1023u);
  const unsigned psm_s = smem_u32(psm);
  uint64_t* bars = reinterpret_cast<uint64_t*>(psm + PSTAGES * STAGE + CBYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + PSTAGES;
  uint64_t* cfull = bars + 2 * PSTAGES;
  uint64_t* cempty = bars + 2 * PSTAGES + 1;
  const unsigned Cs = psm_s + PSTAGES * STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < PSTAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, PCONS); }
    mbar_init(cfull, 1);
    mbar_init(cempty, PCONS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int* tile_ring = reinterpret_cast<int*>(bars + 2 * PSTAGES + 2);
  const long long tiles_per_b = (long long)g.tiles_m * g.tiles_n;
  const int total = (int)(tiles_per_b * g.batch);
  const int ksteps = g.K / PBK;

  if (warp == PCONS) {
    // ---------------- producer warp (one elected lane) ----------------
    // Tiles are claimed from a global counter, so CTAs that start late (SMs
    // busy with kernels of other streams) just take fewer tiles.
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapC) : "memory");
      int stage = 0;
      unsigned phase = 0, cphase = 0;
      for (int seq = 0;; ++seq) {
        const int t = atomicAdd(g.ctr, 1);
        mbar_wait(empty + stage, phase ^ 1);
        tile_ring[seq & (PRING - 1)] = t < total ? t : -1;
        if (t >= total) {  // no tile left: release the consumers
          mbar_arrive(full + stage);
          break;
        }
        const int b = (int)(t / tiles_per_b);
        const int rem = (int)(t % tiles_per_b);
        const int m0 = (rem / g.tiles_n) * PBM, n0 = (rem % g.tiles_n) * BN;
        const int ab = (g.a_bmap ? __ldg(g.a_bmap + b) : b) * g.a_bmul + g.a_badd;
        for (int ks = 0; ks < ksteps; ++ks) {
          if (ks > 0) mbar_wait(empty + stage, phase ^ 1);
          unsigned char* base = psm + stage * STAGE;
          mbar_arrive_expect_tx(full + stage, STAGE);
          const int k0 = ks * PBK;
          tma_load3(base, &mapA, 2 * (g.a_col0 + k0), g.a_row0 + m0, ab, full + stage);
          tma_load3(base + P_A_HALF, &mapA, 2 * (g.a_col0 + k0 + PAK), g.a_row0 + m0, ab, full + stage);
          if constexpr (BSW) {
#pragma unroll
            for (int jb = 0; jb < BN / PAK; ++jb)
              tma_load3(base + P_A_BYTES + jb * P_B_BOX, &mapB, 2 * (g.b_col0 + n0 + jb * PAK), g.b_row0 + k0, b,
                        full + stage);
          } else {
            tma_load3(base + P_A_BYTES, &mapB, 2 * (g.b_col0 + n0), g.b_row0 + k0, b, full + stage);
          }
          if (++stage == PSTAGES) { stage = 0; phase ^= 1; }
        }
        // C block of this tile: requested once the consumers released the
        // previous tile's C, i.e. while this tile's main loop runs
        if (g.beta) {
          mbar_wait(cempty, cphase ^ 1);
          mbar_arrive_expect_tx(cfull, CBYTES);
          tma_load3(psm + PSTAGES * STAGE, &mapC, 2 * (g.c_col0 + n0), g.c_row0 + m0, b, cfull);
          cphase ^= 1;
        }
      }
      // the last CTA out resets the counters for the next launch on this stream
      __threadfence();
      if (atomicAdd(g.ctr + 1, 1) == (int)gridDim.x - 1) {
        g.ctr[0] = 0;
        g.ctr[1] = 0;
        __threadfence();
      }
    }
  } else {
    // ---------------- consumer warps ----------------
    const int wm = (warp / WARPS_N) * (WI * 8), wn = (warp % WARPS_N) * (WJ * 8);
    int stage = 0;
    unsigned phase = 0, cphase = 0;
    for (int seq = 0;; ++seq) {
      // the tile id is published before the first stage of the tile completes
      mbar_wait(full + stage, phase);
      const int t = tile_ring[seq & (PRING - 1)];
      if (t < 0) break;
      const int b = (int)(t / tiles_per_b);
      const int rem = (int)(t % tiles_per_b);
      const int m0 = (rem / g.tiles_n) * PBM, n0 = (rem % g.tiles_n) * BN;
      // two accumulator sets per 8x8 block: re += ar br - ai bi, im += ar bi + ai br
      // (16 independent chains per warp keep the DMMA pipe fed; 64 accumulator
      // registers leave room under the 168-register cap of a 9-warp CTA)
      double are[WI][WJ][2], aim[WI][WJ][2];
#pragma unroll
      for (int i = 0; i < WI; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) are[i][j][h] = aim[i][j][h] = 0.0;
      for (int ks = 0; ks < ksteps; ++ks) {
        mbar_wait(full + stage, phase);
        const unsigned As = psm_s + stage * STAGE;
        const unsigned Bs = As + P_A_BYTES;
#pragma unroll
        for (int ts = 0; ts < PBK / 4; ++ts) {
          cplx af[WI], bf[WJ];
          // DMMA step ts covers k = 8 (ts / 2) + k8, k8 = 2q + (ts % 2) (BSW) or 4 (ts % 2) + q.
          // A element (r, k): box k/8, row r (128 B), 16-B chunk (k%8) ^ (r%8);
          // B element (k, c), BSW: box c/8, row k (128 B), 16-B chunk (c%8) ^ (k%8)
          const int k8 = BSW ? 2 * (lane & 3) + (ts & 1) : 4 * (ts & 1) + (lane & 3);
          const unsigned sw = (unsigned)(k8 ^ (lane >> 2)) << 4;
#pragma unroll
          for (int j = 0; j < WJ; ++j)
            bf[j] = BSW ? lds_c(Bs + ((wn + j * 8) / PAK) * P_B_BOX + ((ts >> 1) * 8 + k8) * 128 + sw)
                        : lds_c(Bs + (((ts >> 1) * 8 + k8) * BN + wn + j * 8 + (lane >> 2)) * 16);
#pragma unroll
          for (int i = 0; i < WI; ++i)
            af[i] = lds_c(As + (ts >> 1) * P_A_HALF + (wm + i * 8 + (lane >> 2)) * 128 + sw);
#pragma unroll
          for (int i = 0; i < WI; ++i)
#pragma unroll
            for (int j = 0; j < WJ; ++j) {
              dmma884(are[i][j][0], are[i][j][1], af[i].x, bf[j].x);
              dmma884(aim[i][j][0], aim[i][j][1], af[i].x, bf[j].y);
            }
#pragma unroll
          for (int i = 0; i < WI; ++i) {
            const double nai = -af[i].y;
#pragma unroll
            for (int j = 0; j < WJ; ++j) {
              dmma884(are[i][j][0], are[i][j][1], nai, bf[j].y);
              dmma884(aim[i][j][0], aim[i][j][1], af[i].y, bf[j].x);
            }
          }
        }
        // The stage is refilled by TMA (async proxy) once every warp arrived:
        // order this warp's shared-memory reads before that write.  Without the
        // fence the arrive can overtake a still-pending LDS (ptxas schedules it
        // ahead of the last DMMAs), which corrupts tiles when the SM's shared
        // memory pipe is slowed by co-resident CTAs of other streams.
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + stage);
        if (++stage == PSTAGES) { stage = 0; phase ^= 1; }
      }
      // epilogue: C - acc (or +acc when beta == 0), straight to global
      if (g.beta) {
        mbar_wait(cfull, cphase);
        cphase ^= 1;
      }
      cplx* Cb = g.C + (long long)b * g.sC;
#pragma unroll
      for (int i = 0; i < WI; ++i) {
        const int rl = wm + i * 8 + (lane >> 2);
        const int r = m0 + rl;
#pragma unroll
        for (int j = 0; j < WJ; ++j) {
          const int cl = wn + j * 8 + 2 * (lane & 3);
          const int c = n0 + cl;
          if (r < g.M) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (c + h < g.N) {
                const double pr = are[i][j][h], pi = aim[i][j][h];
                cplx outv;
                if (g.beta) {
                  const cplx v = lds_c(Cs + (rl * BN + cl + h) * 16);
                  outv = cmk(v.x - pr, v.y - pi);
                } else {
                  outv = cmk(pr, pi);
                }
                Cb[(long long)(g.c_row0 + r) * g.ldc + g.c_col0 + c + h] = outv;
              }
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (g.beta && lane == 0) mbar_arrive(cempty);
    }

  }
}

// Encode a TMA map over a batch of row-major complex128 matrices viewed as a
// float64 tensor {2*cols, rows, batch}, with a box of box_rows x box_cols
// complex elements.  Out-of-range boxes are zero-filled by the hardware.
static inline int encode_c128_map(CUtensorMap* map, const cplx* base, int cols, int rows, int batch, long long ld,
                           long long bstride, int box_cols, int box_rows, bool swizzle128 = false) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return (int)cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return (int)cudaErrorInvalidValue;
  cuuint64_t dims[3] = {(cuuint64_t)2 * cols, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 16, (cuuint64_t)(bstride > 0 ? bstride : ld * rows) * 16};
  cuuint32_t estr[3] = {1, 1, 1};
  cuuint32_t box[3] = {(cuuint32_t)(2 * box_cols), (cuuint32_t)box_rows, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<cplx*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE,
                      swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

// A-operand map: 64 x 8 boxes with the 128-byte swizzle (two per K slice).
static inline int encode_a_map(CUtensorMap* map, const cplx* base, int cols, int rows, int batch, long long ld,
                               long long bstride) {
  return encode_c128_map(map, base, cols, rows, batch, ld, bstride, PAK, PBM, true);
}

// B-operand map of the solves: 16 x 8 boxes with the 128-byte swizzle (BSW).
static inline int encode_b_swz_map(CUtensorMap* map, const cplx* base, int cols, int rows, int batch, long long ld,
                                   long long bstride) {
  return encode_c128_map(map, base, cols, rows, batch, ld, bstride, PAK, PBK, true);
}

// Tile width for a right-hand-side block of K columns: the smallest padded
// width ceil(K / bn) * bn weighted by the measured efficiency of each tile
// shape (n = 4096, 128 pencils, padded TF/s relative to the 64-wide tile;
// tools/solve_bn_sweep.sh).  Unswizzled B (BSW off) the narrow tiles were
// shared-memory bound (56: 0.87, 48: 0.87, 40: 0.876, 32: 0.93); with the
// swizzled boxes every width runs within 2.5 % of the 64-wide tile, so
// K = 118 takes 3 x 40 (62.0 ms per pass vs 65.3 ms as 2 x 64), K = 110
// 2 x 56 (58.6 vs 65.2 ms) and K = 32 one 32-wide tile.
static inline int pick_tile_n(int K, bool bswz = true) {
  const int cand[5] = {64, 56, 48, 40, 32};
  const double eff_plain[5] = {1.0, 0.87, 0.87, 0.876, 0.93};
  const double eff_swz[5] = {1.0, 0.976, 0.997, 0.99, 0.997};
  const double* eff = bswz ? eff_swz : eff_plain;
  int best = 64;
  double cost = (K + 63) / 64 * 64;
  for (int i = 1; i < 5; ++i) {
    const double w = (double)((K + cand[i] - 1) / cand[i] * cand[i]) / eff[i];
    if (w < cost) { best = cand[i]; cost = w; }
  }
  return best;
}

// Maps for the three operand roles: A (64 x 8 swizzled boxes), B (16 x 64), C (64 x 64).
struct OperandMaps {
  CUtensorMap a, b, c;
};
using PencilMaps = OperandMaps;

static inline int encode_pencil_maps(PencilMaps& pm, cplx* base, int n, long long ld, long long pstride, int batch) {
  CIRR_TRY(encode_a_map(&pm.a, base, n, n, batch, ld, pstride));
  CIRR_TRY(encode_c128_map(&pm.b, base, n, n, batch, ld, pstride, PBN, PBK));
  CIRR_TRY(encode_c128_map(&pm.c, base, n, n, batch, ld, pstride, PBN, PBM));
  return 0;
}

// C[b] -= A[b] @ B[b] (beta = 1) or C[b] = A[b] @ B[b] (beta = 0) on sub-blocks addressed through TMA maps (A: mapA with
// origin (a_row0, a_col0), etc.); C is also written through (C, ldc, sC).
// K is rounded up to a multiple of 16: the extra slice must lie outside the
// tensors (zero-filled) or hold zeros.
static inline int zgemm_sub_maps(const CUtensorMap& mapA, const CUtensorMap& mapB, const CUtensorMap& mapC, int M, int N,
                          int K, int batch, int a_row0, int a_col0, int b_row0, int b_col0, int c_row0, int c_col0,
                          cplx* C, long long ldc, long long sC, cudaStream_t stream, int beta = 1,
                          int a_bmul = 1, int a_badd = 0, const int* a_bmap = nullptr, int bn = PBN,
                          bool bswz = false) {
  if (M <= 0 || N <= 0 || K <= 0 || batch <= 0) return 0;
  static bool attr = false;
  static int sms = 0;
  if (!attr) {
    cudaFuncSetAttribute(zgemm_sub_tma<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<64>::SMEM);
    cudaFuncSetAttribute(zgemm_sub_tma<56, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<56>::SMEM);
    cudaFuncSetAttribute(zgemm_sub_tma<48, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<48>::SMEM);
    cudaFuncSetAttribute(zgemm_sub_tma<40, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<40>::SMEM);
    cudaFuncSetAttribute(zgemm_sub_tma<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<32>::SMEM);
    cudaFuncSetAttribute(zgemm_sub_tma<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<64>::SMEM);
    cudaFuncSetAttribute(zgemm_sub_tma<56, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<56>::SMEM);
    cudaFuncSetAttribute(zgemm_sub_tma<48, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<48>::SMEM);
    cudaFuncSetAttribute(zgemm_sub_tma<40, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<40>::SMEM);
    cudaFuncSetAttribute(zgemm_sub_tma<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TileBytes<32>::SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  const int Kr = (K + PBK - 1) / PBK * PBK;
  int* ctr = cirr_tile_counter(stream);
  if (!ctr) return (int)cudaErrorMemoryAllocation;
  SubGemmGeom g{M, N, Kr, batch, a_row0, a_col0, b_row0, b_col0, c_row0, c_col0, C, ldc, sC,
                (M + PBM - 1) / PBM, (N + bn - 1) / bn, beta, a_bmul, a_badd, ctr, a_bmap};
  const long long tiles = (long long)g.tiles_m * g.tiles_n * batch;
  // persistent grid: every SM, or fewer when cirr_set_gemm_ctas leaves SMs to
  // latency-bound kernels on other streams (the dynamic tile scheduler adapts)
  const int cap = (g_cirr_gemm_cap > 0 && g_cirr_gemm_cap < sms) ? g_cirr_gemm_cap : sms;
  const int grid = (int)(tiles < cap ? tiles : cap);
#define CIRR_SUB_TMA(BNV, SW) \
  zgemm_sub_tma<BNV, SW><<<grid, PTHREADS, TileBytes<BNV>::SMEM, stream>>>(mapA, mapB, mapC, g)
  switch (bn * 2 + (bswz ? 1 : 0)) {
    case 128: CIRR_SUB_TMA(64, false); break;
    case 112: CIRR_SUB_TMA(56, false); break;
    case 96: CIRR_SUB_TMA(48, false); break;
    case 80: CIRR_SUB_TMA(40, false); break;
    case 64: CIRR_SUB_TMA(32, false); break;
    case 129: CIRR_SUB_TMA(64, true); break;
    case 113: CIRR_SUB_TMA(56, true); break;
    case 97: CIRR_SUB_TMA(48, true); break;
    case 81: CIRR_SUB_TMA(40, true); break;
    case 65: CIRR_SUB_TMA(32, true); break;
    default: return (int)cudaErrorInvalidValue;
  }
#undef CIRR_SUB_TMA
  cirr_note_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

// A22 -= L21 U12 for panel step (k, jb) of every pencil, via the TMA kernel.
static inline int lu_update_tma(const PencilMaps& pm, cplx* pencils, int n, long long ld, long long pstride, int batch,
                         int k, int jb, cudaStream_t stream) {
  const int rest = n - k - jb;
  return zgemm_sub_maps(pm.a, pm.b, pm.c, rest, rest, jb, batch, k + jb, k, k, k + jb, k + jb, k + jb, pencils, ld,
                        pstride, stream);
}

}  // namespace cirr
