// Experiment (round 2, last session): Ozaki-scheme int8 slice products on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in TMEM) as a
// possible replacement for the DMMA trailing update.  Standalone: checks the
// slice-product accumulators acc_d = sum_{p+q=d} A_p B_q^T against the host and
// times the kernel at the LU's trailing-update shape.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 tools/i8_umma.cu -o tools/i8_umma -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

constexpr int BM = 128;      // accumulator rows = TMEM lanes
constexpr int BN = 64;       // accumulator columns (real)
constexpr int KB = 64;       // bytes of K per stage (64-byte swizzle rows)
constexpr int NSTAGE = 2;
constexpr int THREADS = 192; // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue

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
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}
// K-major operand tile with the 64-byte swizzle: rows of 64 bytes, groups of 8
// rows 512 bytes apart (SBO), descriptor version 1 (Blackwell), layout type 4.
__device__ __forceinline__ uint64_t umma_desc_sw64(unsigned saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;        // stride byte offset
  d |= (uint64_t)1 << 46;                 // version
  d |= (uint64_t)4 << 61;                 // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ void umma_i8(unsigned tmem_d, uint64_t da, uint64_t db, unsigned idesc, unsigned acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}"
      ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld16(unsigned taddr, unsigned* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr) : "memory");
}

struct Geom {
  int M, N, K;      // rows of A, rows of B (real output columns), bytes of K
  int S;            // slices
  int tiles_m, tiles_n;
  int* acc;         // [S][M][N] int32 dump (check mode) or nullptr
  long long* sink;  // timing mode: one value per CTA so the epilogue is not dead
};

template <int S>
__global__ void __launch_bounds__(THREADS, 1) ozaki_i8_kernel(const __grid_constant__ CUtensorMap mapA,
                                                               const __grid_constant__ CUtensorMap mapB, Geom g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int A_SLICE = BM * KB, B_SLICE = BN * KB;
  constexpr int STAGE = S * (A_SLICE + B_SLICE);
  uint64_t* full = (uint64_t*)(smem + NSTAGE * STAGE);
  uint64_t* empty = full + NSTAGE;
  uint64_t* tfull = empty + NSTAGE;
  uint64_t* tempty = tfull + 1;
  unsigned* tmem_slot = (unsigned*)(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = *tmem_slot;

  const int ntiles = g.tiles_m * g.tiles_n;
  const int nkb = g.K / KB;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t / g.tiles_n) * BM, n0 = (t % g.tiles_n) * BN;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int st = it % NSTAGE;
          const unsigned ph = (it / NSTAGE) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], STAGE);
          uint8_t* base = smem + st * STAGE;
#pragma unroll
          for (int s = 0; s < S; ++s) {
            tma_load3(base + s * A_SLICE, &mapA, kb * KB, m0, s, &full[st]);
            tma_load3(base + S * A_SLICE + s * B_SLICE, &mapB, kb * KB, n0, s, &full[st]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(BN >> 3) << 17) | ((unsigned)(BM >> 4) << 24);
      int it = 0, tl = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
        mbar_wait(tempty, (tl & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int st = it % NSTAGE;
          const unsigned ph = (it / NSTAGE) & 1;
          mbar_wait(&full[st], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const unsigned abase = smem_u32(smem + st * STAGE), bbase = abase + S * A_SLICE;
#pragma unroll
          for (int ks = 0; ks < KB / 32; ++ks) {
#pragma unroll
            for (int d = 0; d < S; ++d) {
#pragma unroll
              for (int p = 0; p <= d; ++p) {
                const int q = d - p;
                const uint64_t da = umma_desc_sw64(abase + p * A_SLICE + ks * 32);
                const uint64_t db = umma_desc_sw64(bbase + q * B_SLICE + ks * 32);
                umma_i8(tmem + d * BN, da, db, idesc, (kb > 0 || ks > 0 || p > 0) ? 1u : 0u);
              }
            }
          }
          umma_commit(&empty[st]);
        }
        umma_commit(tfull);
      }
    }
  } else {
    const int quad = warp & 3;  // TMEM lanes 32*quad .. 32*quad+31
    int tl = 0;
    long long sink = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
      const int m0 = (t / g.tiles_n) * BM, n0 = (t % g.tiles_n) * BN;
      mbar_wait(tfull, tl & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m0 + quad * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        long long hi[16], lo[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) hi[j] = lo[j] = 0;
#pragma unroll
        for (int d = 0; d < S; ++d) {
          unsigned v[16];
          tmem_ld16(tmem + ((unsigned)(quad * 32) << 16) + d * BN + c, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (g.acc) {
            if (row < g.M)
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (n0 + c + j < g.N) g.acc[((size_t)d * g.M + row) * g.N + n0 + c + j] = (int)v[j];
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (d < 4) hi[j] = (hi[j] << 7) + (int)v[j];
            else lo[j] = (lo[j] << 7) + (int)v[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) sink += hi[j] ^ lo[j];
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
    if (g.sink) g.sink[blockIdx.x * 128 + (warp - 2) * 32 + lane] = sink;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}
// slices [S][rows][K] int8, box {KB, box_rows, 1}, 64-byte swizzle
static void make_map(CUtensorMap* map, const int8_t* base, int K, int rows, int S, int box_rows) {
  static auto encode = get_encode();
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)S};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)K * rows};
  cuuint32_t box[3] = {(cuuint32_t)KB, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("cuTensorMapEncodeTiled failed: %d\n", (int)r); exit(1); }
}

template <int S>
static int run(int M, int N, int K, bool check, int reps) {
  std::vector<int8_t> hA((size_t)S * M * K), hB((size_t)S * N * K);
  uint32_t seed = 12345u;
  auto rnd = [&]() { seed = seed * 1664525u + 1013904223u; return (int)((seed >> 16) % 129) - 64; };
  for (auto& v : hA) v = (int8_t)rnd();
  for (auto& v : hB) v = (int8_t)rnd();
  int8_t *dA, *dB;
  CK(cudaMalloc(&dA, hA.size()));
  CK(cudaMalloc(&dB, hB.size()));
  CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  CUtensorMap mA, mB;
  make_map(&mA, dA, K, M, S, BM);
  make_map(&mB, dB, K, N, S, BN);
  Geom g{};
  g.M = M; g.N = N; g.K = K; g.S = S;
  g.tiles_m = (M + BM - 1) / BM;
  g.tiles_n = (N + BN - 1) / BN;
  int* dacc = nullptr;
  long long* dsink = nullptr;
  if (check) { CK(cudaMalloc(&dacc, (size_t)S * M * N * 4)); CK(cudaMemset(dacc, 0xff, (size_t)S * M * N * 4)); }
  CK(cudaMalloc(&dsink, 148 * 128 * 8));
  g.acc = dacc; g.sink = dsink;
  const int smem = NSTAGE * S * (BM * KB + BN * KB) + 1024 + 256;
  CK(cudaFuncSetAttribute(ozaki_i8_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int grid = g.tiles_m * g.tiles_n < 148 ? g.tiles_m * g.tiles_n : 148;
  ozaki_i8_kernel<S><<<grid, THREADS, smem>>>(mA, mB, g);
  CK(cudaDeviceSynchronize());
  int bad = 0;
  if (check) {
    std::vector<int> hacc((size_t)S * M * N);
    CK(cudaMemcpy(hacc.data(), dacc, hacc.size() * 4, cudaMemcpyDeviceToHost));
    for (int d = 0; d < S; ++d)
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
          long long ref = 0;
          for (int p = 0; p <= d; ++p) {
            const int8_t* a = &hA[((size_t)p * M + i) * K];
            const int8_t* b = &hB[((size_t)(d - p) * N + j) * K];
            for (int k = 0; k < K; ++k) ref += (int)a[k] * (int)b[k];
          }
          if ((long long)hacc[((size_t)d * M + i) * N + j] != ref) {
            if (bad < 8) printf("  mismatch d=%d i=%d j=%d got %d want %lld\n", d, i, j, hacc[((size_t)d * M + i) * N + j], ref);
            ++bad;
          }
        }
    printf("check S=%d M=%d N=%d K=%d: %s (%d mismatches)\n", S, M, N, K, bad ? "FAIL" : "ok", bad);
  } else {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) ozaki_i8_kernel<S><<<grid, THREADS, smem>>>(mA, mB, g);
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    const double macs = 0.5 * S * (S + 1) * (double)M * N * K;
    // equivalent complex GEMM: m = M, n = N/2, k = K/2
    const double zflops = 8.0 * M * (N / 2.0) * (K / 2.0);
    printf("time S=%d M=%d N=%d K=%d: %.3f ms, %.2f int8 POPS, FP64-equivalent complex GEMM %.1f TF/s (DMMA path ~35.6)\n",
           S, M, N, K, ms, 2 * macs / ms * 1e-12, zflops / ms * 1e-9);
  }
  cudaFree(dA); cudaFree(dB); if (dacc) cudaFree(dacc); cudaFree(dsink);
  return bad;
}

int main(int argc, char** argv) {
  int bad = 0;
  bad += run<1>(128, 64, 64, true, 0);
  bad += run<1>(256, 128, 256, true, 0);
  bad += run<3>(256, 192, 256, true, 0);
  bad += run<8>(384, 128, 512, true, 0);
  if (bad) { printf("FAILED\n"); return 1; }
  run<8>(3584, 7168, 1024, false, 5);
  run<7>(3584, 7168, 1024, false, 5);
  run<1>(3584, 7168, 8192, false, 5);
  return 0;
}
