// gemm.cu — the tensor-core member of the suite: C = A Bt^T, A and Bt N x N bf16 K-major,
// fp32 accumulation in TMEM, bf16 output (R-17).  Tensor bound: 2N^3 FLOPs.
//
// sm_100a design, hand-written PTX (no CUTLASS).  B >= 192: CTA pairs (cta_group::2, 256 x 256
// tiles, below); B = 128/160 (too few warps for the split roles): one CTA per 128 x 256 tile:
//   warp 0, one lane : TMA producer — cp.async.bulk.tensor 2D loads of the A (128 x 64) and
//                      Bt (256 x 64) K-slices, 128-byte swizzle, into a kStages-deep ring of
//                      shared-memory stages guarded by full/empty mbarriers;
//   warp 1, one lane : MMA issuer — four tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256,
//                      K=16) per stage into a 256-column fp32 TMEM accumulator, tcgen05.commit
//                      releases the stage back to the producer;
//   all warps        : epilogue — tcgen05.ld 32 lanes x 32 columns per warp (lane quadrant
//                      = warp % 4), convert to bf16, store 64 contiguous bytes per row.
// The block size of the sweep sets how many warps share the epilogue; fewer than 128 threads
// cannot cover the four TMEM lane quadrants, so those points are INVALID_CONFIG rows (the
// paper's NaN rows for configurations a kernel does not support).
// Requires N % 8 == 0 (TMA row pitch must be a multiple of 16 bytes).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kern_common.cuh"

namespace lscat {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, UK = 16;
constexpr int kStages = 4;
constexpr int kGroupM = 16;  // tile rows per rasterisation group
constexpr int kStageA = BM * BK * 2;  // 16 KB
constexpr int kStageB = BN * BK * 2;  // 32 KB
constexpr int kSmem = kStages * (kStageA + kStageB) + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t kTmemCols = 256;

struct GemmMaps {
  CUtensorMap a, b;  // A: 128-row boxes; Bt: 256-row boxes (one CTA's 128 x 256 tile)
  CUtensorMap b128;  // Bt: 128-row boxes (the 2-CTA kernel: each CTA of a pair loads half of B)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// K-major, 128-byte swizzle smem matrix descriptor (SBO = 1024 B between 8-row groups).
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;             // start address
  d |= (uint64_t)1 << 16;                   // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;         // stride byte offset
  d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, M = 128, N = 256.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

template <int B>
__global__ void __launch_bounds__(B, 1) gemm_kernel(const __grid_constant__ GemmMaps maps,
                                                    __nv_bfloat16* __restrict__ C, int N) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kStageA;
  uint64_t* full = (uint64_t*)(sB + kStages * kStageB);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = (uint32_t*)(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterisation: consecutive CTAs walk kGroupM tile rows before the next tile
  // column, so a wave's A and Bt tiles stay L2-resident (A is re-read once per group, not per
  // tile column)
  const int mt = (N + BM - 1) / BM, nt = (N + BN - 1) / BN;
  const int pid = blockIdx.x, per_group = kGroupM * nt;
  const int first_m = (pid / per_group) * kGroupM;
  const int gm = min(mt - first_m, kGroupM);
  const int m0 = (first_m + (pid % per_group) % gm) * BM;
  const int n0 = ((pid % per_group) / gm) * BN;
  const int kblocks = (N + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.b) : "memory");
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    for (int kb = 0; kb < kblocks; kb++) {
      const int s = kb % kStages;
      const uint32_t ph = (kb / kStages) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], kStageA + kStageB);
      tma_load_2d(sA + s * kStageA, &maps.a, &full[s], kb * BK, m0);
      tma_load_2d(sB + s * kStageB, &maps.b, &full[s], kb * BK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    for (int kb = 0; kb < kblocks; kb++) {
      const int s = kb % kStages;
      const uint32_t ph = (kb / kStages) & 1;
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t ad = sw128_desc(sA + s * kStageA), bd = sw128_desc(sB + s * kStageB);
#pragma unroll
      for (int k = 0; k < BK / UK; k++) {
        // advance the start address by k * 32 bytes inside the 128-byte swizzle atom
        mma_bf16(tmem, ad + (uint64_t)(k * UK * 2 >> 4), bd + (uint64_t)(k * UK * 2 >> 4),
                 (kb | k) != 0);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(tmem_full);
  }
  __syncwarp();

  // ---- epilogue: every warp, lane quadrant q = warp % 4, 32-column chunks round-robin
  mbar_wait(tmem_full, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  constexpr int W = B / 32;
  const int q = warp & 3;
  const int nq = (W - q + 3) / 4;      // warps sharing quadrant q
  const int iq = warp >> 2;            // this warp's index among them
  const int row = m0 + q * 32 + lane;
  for (int c = iq; c < BN / 32; c += nq) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int col = n0 + c * 32;
    if (row < N && col < N) {
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; i++) {
        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        pk[i] = *reinterpret_cast<uint32_t*>(&h);
      }
      __nv_bfloat16* dst = C + (size_t)row * N + col;
      if (col + 32 <= N) {
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int i = 0; i < 4; i++) d4[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      } else {
        for (int i = 0; i < 32 && col + i < N; i++) {
          uint32_t w = pk[i >> 1];
          uint16_t h = (i & 1) ? (uint16_t)(w >> 16) : (uint16_t)(w & 0xFFFF);
          reinterpret_cast<uint16_t*>(dst)[i] = h;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                 : "memory");
  }
}

// Persistent variant (B >= 192: two role warps + at least four epilogue warps).  One CTA per
// SM walks the output tiles blockIdx.x, blockIdx.x + gridDim.x, ... (grouped raster order):
//   warp 0, one lane : TMA producer over the continuous (tile, k-block) sequence;
//   warp 1, one lane : MMA issuer; tile j accumulates into TMEM buffer j & 1 (2 x 256 of the
//                      512 columns), waiting on tmem_empty[j & 1] before the first k-block;
//   warps 2..W-1     : epilogue of tile j from buffer j & 1 while the MMA already runs tile
//                      j + 1 in the other buffer; each warp arrives on tmem_empty once its
//                      tcgen05.ld of the tile are done.
// So the tensor pipe is not idle during the epilogue and the per-tile prologue (barrier init,
// TMEM allocation) is paid once per CTA.  Measured at N = 8192 in the burst regime
// (scripts/gemm_ab.py, interleaved short bursts): 738 us = 1489 TFLOP/s (B = 192) vs 767 us =
// 1433 TFLOP/s for the one-tile-per-CTA kernel (B = 128).
constexpr uint32_t kTmemColsP = 512;

template <int B>
__global__ void __launch_bounds__(B, 1) gemm_persistent_kernel(const __grid_constant__ GemmMaps maps,
                                                               __nv_bfloat16* __restrict__ C, int N) {
  constexpr int W = B / 32;
  static_assert(W >= 6, "persistent GEMM needs 2 role warps + 4 epilogue warps");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kStageA;
  uint64_t* full = (uint64_t*)(sB + kStages * kStageB);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;   // [2]
  uint32_t* tmem_slot = (uint32_t*)(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = (N + BM - 1) / BM, nt = (N + BN - 1) / BN, ntiles = mt * nt;
  const int per_group = kGroupM * nt;
  const int kblocks = (N + BK - 1) / BK;
  auto tile_origin = [&](int t, int& m0, int& n0) {
    const int first_m = (t / per_group) * kGroupM;
    const int gm = min(mt - first_m, kGroupM);
    m0 = (first_m + (t % per_group) % gm) * BM;
    n0 = ((t % per_group) / gm) * BN;
  };

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.b) : "memory");
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], W - 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemColsP)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      uint32_t it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m0, n0;
        tile_origin(t, m0, n0);
        for (int kb = 0; kb < kblocks; kb++, it++) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], kStageA + kStageB);
          tma_load_2d(sA + s * kStageA, &maps.a, &full[s], kb * BK, m0);
          tma_load_2d(sB + s * kStageB, &maps.b, &full[s], kb * BK, n0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      uint32_t it = 0, j = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, j++) {
        const uint32_t buf = j & 1, use = j >> 1;
        mbar_wait(&tmem_empty[buf], (use & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + buf * BN;
        for (int kb = 0; kb < kblocks; kb++, it++) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = sw128_desc(sA + s * kStageA), bd = sw128_desc(sB + s * kStageB);
#pragma unroll
          for (int k = 0; k < BK / UK; k++)
            mma_bf16(acc, ad + (uint64_t)(k * UK * 2 >> 4), bd + (uint64_t)(k * UK * 2 >> 4), (kb | k) != 0);
          mma_commit(&empty[s]);
        }
        mma_commit(&tmem_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue warps: lane quadrant q = warp % 4 (the TMEM lanes this warp may access);
    // the warps of one quadrant split the 8 32-column chunks
    const int q = warp & 3;
    const int first_w = q >= 2 ? q : q + 4;  // first epilogue warp (>= 2) of quadrant q
    const int iq = (warp - first_w) >> 2;
    const int nq = (W - 1 - first_w) / 4 + 1;
    uint32_t j = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, j++) {
      int m0, n0;
      tile_origin(t, m0, n0);
      const uint32_t buf = j & 1, use = j >> 1;
      mbar_wait(&tmem_full[buf], use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m0 + q * 32 + lane;
      for (int c = iq; c < BN / 32; c += nq) {
        uint32_t v[32];
        const uint32_t taddr = tmem + buf * BN + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
              "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
              "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int col = n0 + c * 32;
        if (row < N && col < N) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; i++) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
            pk[i] = *reinterpret_cast<uint32_t*>(&h);
          }
          __nv_bfloat16* dst = C + (size_t)row * N + col;
          if (col + 32 <= N) {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
            for (int i = 0; i < 4; i++) d4[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          } else {
            for (int i = 0; i < 32 && col + i < N; i++) {
              uint32_t w = pk[i >> 1];
              uint16_t h = (i & 1) ? (uint16_t)(w >> 16) : (uint16_t)(w & 0xFFFF);
              reinterpret_cast<uint16_t*>(dst)[i] = h;
            }
          }
        }
      }
      // this warp's reads of buffer `buf` are complete: hand it back to the MMA issuer
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[buf])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemColsP)
                 : "memory");
  }
}

// CTA-pair variant (B >= 192, cluster of 2): the pair computes a 256 x 256 output tile with
// tcgen05.mma.cta_group::2 (M = 256: 128 rows in each CTA's TMEM).  The default for B >= 192;
// measured at N = 8192 in the burst regime (scripts/gemm_ab.py): 716 us = 1535 TFLOP/s (0.95
// of cuBLAS burst) vs 756 us for the one-CTA persistent kernel in the same run.  Each CTA loads its own
// 128 rows of A and its own 128 columns of B per k-block (32 KB per stage instead of 48 KB:
// half the B traffic per SM), 7-stage ring (4 / 5 / 6 / 7 stages: 1500 / 1543 / 1543 / 1563
// TFLOP/s at N = 8192, scripts/gemm_variants.sh).  Both CTAs' TMA loads complete on the leader
// CTA's full barrier (cta_group::2 TMA, peer bit cleared); the leader's single MMA thread
// issues the pair's MMAs and commits with a multicast arrive to both CTAs' empty / tmem_full
// barriers; every epilogue warp of both CTAs arrives on the leader's tmem_empty barrier.
// Persistent over tiles with two TMEM accumulators (2 x 256 columns per CTA).
#ifndef GEMM2_STAGES
#define GEMM2_STAGES 7
#endif
constexpr int kStages2 = GEMM2_STAGES;  // calibration switch (scripts/gemm_variants.sh)
#ifndef GEMM2_GROUPM
#define GEMM2_GROUPM 8
#endif
constexpr int kGroupM2 = GEMM2_GROUPM;  // 256-row tile rows per raster group: 4 / 8 / 16 / 32 ->
                                        // 1539 / 1584 / 1569 / 1488 TFLOP/s (scripts/gemm_variants2.sh)
constexpr int kStage2A = 128 * BK * 2, kStage2B = 128 * BK * 2;  // 16 KB each
constexpr int kSmem2 = kStages2 * (kStage2A + kStage2B) + 1024 + 256;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address -> the leader CTA's copy
// kind::f16, D fp32, A/B bf16 K-major, M = 256 (the pair), N = 256
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

template <int B>
__global__ void __launch_bounds__(B, 1) gemm_2cta_kernel(const __grid_constant__ GemmMaps maps,
                                                         __nv_bfloat16* __restrict__ C, int N) {
  constexpr int W = B / 32;
  static_assert(W >= 6, "2-CTA GEMM needs 2 role warps + 4 epilogue warps");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages2 * kStage2A;
  uint64_t* full = (uint64_t*)(sB + kStages2 * kStage2B);
  uint64_t* empty = full + kStages2;
  uint64_t* tmem_full = empty + kStages2;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;    // [2] (the leader's are used)
  uint32_t* tmem_slot = (uint32_t*)(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  constexpr int TM = 256, TN = 256;
  const int mt = (N + TM - 1) / TM, nt = (N + TN - 1) / TN, ntiles = mt * nt;
  const int per_group = kGroupM2 * nt;
  const int kblocks = (N + BK - 1) / BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  auto tile_origin = [&](int t, int& m0, int& n0) {
    const int first_m = (t / per_group) * kGroupM2;
    const int gm = min(mt - first_m, kGroupM2);
    m0 = (first_m + (t % per_group) % gm) * TM;
    n0 = ((t % per_group) / gm) * TN;
  };

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.b128) : "memory");
    for (int s = 0; s < kStages2; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 2 * (W - 2));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemColsP)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs): own A rows, own B columns
      uint32_t it = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        int m0, n0;
        tile_origin(t, m0, n0);
        for (int kb = 0; kb < kblocks; kb++, it++) {
          const int s = it % kStages2;
          const uint32_t ph = (it / kStages2) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          const uint32_t fb = smem_u32(&full[s]) & kPeerMask;  // the leader's full barrier
          if (leader)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                         "r"(2 * (kStage2A + kStage2B))
                         : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(sA + s * kStage2A)),
              "l"(&maps.a), "r"(fb), "r"(kb * BK), "r"(m0 + 128 * (int)rank)
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(sB + s * kStage2B)),
              "l"(&maps.b128), "r"(fb), "r"(kb * BK), "r"(n0 + 128 * (int)rank)
              : "memory");
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ---- MMA issuer (leader CTA only)
      uint32_t it = 0, j = 0;
      for (int t = pair; t < ntiles; t += npairs, j++) {
        const uint32_t buf = j & 1, use = j >> 1;
        mbar_wait(&tmem_empty[buf], (use & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + buf * TN;
        for (int kb = 0; kb < kblocks; kb++, it++) {
          const int s = it % kStages2;
          const uint32_t ph = (it / kStages2) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = sw128_desc(sA + s * kStage2A), bd = sw128_desc(sB + s * kStage2B);
#pragma unroll
          for (int k = 0; k < BK / UK; k++) {
            const uint64_t a2 = ad + (uint64_t)(k * UK * 2 >> 4), b2 = bd + (uint64_t)(k * UK * 2 >> 4);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc),
                "l"(a2), "l"(b2), "r"(kIdesc2), "r"((kb | k) != 0 ? 1 : 0));
          }
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&empty[s])),
              "h"((uint16_t)3)
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&tmem_full[buf])),
            "h"((uint16_t)3)
            : "memory");
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue warps (both CTAs): this CTA's 128 rows of the pair's tile
    const int q = warp & 3;
    const int first_w = q >= 2 ? q : q + 4;
    const int iq = (warp - first_w) >> 2;
    const int nq = (W - 1 - first_w) / 4 + 1;
    const uint32_t lead_empty = mapa_shared(smem_u32(&tmem_empty[0]), 0);
    uint32_t j = 0;
    for (int t = pair; t < ntiles; t += npairs, j++) {
      int m0, n0;
      tile_origin(t, m0, n0);
      const uint32_t buf = j & 1, use = j >> 1;
      mbar_wait(&tmem_full[buf], use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m0 + 128 * (int)rank + q * 32 + lane;
      for (int c = iq; c < TN / 32; c += nq) {
        uint32_t v[32];
        const uint32_t taddr = tmem + buf * TN + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
              "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
              "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int col = n0 + c * 32;
        if (row < N && col < N) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; i++) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
            pk[i] = *reinterpret_cast<uint32_t*>(&h);
          }
          __nv_bfloat16* dst = C + (size_t)row * N + col;
          if (col + 32 <= N) {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
            for (int i = 0; i < 4; i++) d4[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          } else {
            for (int i = 0; i < 32 && col + i < N; i++) {
              uint32_t w = pk[i >> 1];
              uint16_t h = (i & 1) ? (uint16_t)(w >> 16) : (uint16_t)(w & 0xFFFF);
              reinterpret_cast<uint16_t*>(dst)[i] = h;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(lead_empty + buf * 8)
                     : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the leader's MMAs read both CTAs' smem: nobody leaves early
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemColsP)
                 : "memory");
  }
}

template <int B>
struct GemmL {
  static constexpr bool kSupported = B >= 128;
  // the kernel the default launch runs: CTA pairs for B >= 192 (N % 8 == 0), one tile per CTA
  // for 128 / 160 threads
  static cudaError_t attrs(const void** f, size_t* sm) {
    if constexpr (B >= 192) return kernel_attrs(gemm_2cta_kernel<B>, kSmem2, f, sm);
    else if constexpr (B >= 128) return kernel_attrs(gemm_kernel<B>, kSmem, f, sm);
    else return cudaErrorInvalidConfiguration;
  }
  static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
    if constexpr (B >= 128) {
      const SuiteEntry& e = *a.e;
      // kernel attributes: set once per process (thread-safe one-time initialisation; the
      // value is the same for every sm_100a device)
      static const cudaError_t attr =
          cudaFuncSetAttribute(gemm_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
      if (attr != cudaSuccess) return attr;
      const int sms = a.sms > 0 ? a.sms : 148;
      const int N = (int)e.n;
      const int tiles = ((N + BM - 1) / BM) * ((N + BN - 1) / BN);
      if constexpr (B >= 192) {
        static const int two_cta = [] {  // LSCAT_GEMM_2CTA=0: the one-CTA persistent kernel
          const char* v = getenv("LSCAT_GEMM_2CTA");
          return v ? atoi(v) : 1;
        }();
        if (two_cta && N % 8 == 0) {  // CTA pairs (cluster of 2), persistent
          static const cudaError_t attr2 =
              cudaFuncSetAttribute(gemm_2cta_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2);
          if (attr2 != cudaSuccess) return attr2;
          const int pairs = std::max(1, sms / 2);
          const int tiles2 = ((N + 255) / 256) * ((N + 255) / 256);
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(2 * std::min(tiles2, pairs));
          cfg.blockDim = dim3(B);
          cfg.dynamicSmemBytes = kSmem2;
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = 2;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          return cudaLaunchKernelEx(&cfg, gemm_2cta_kernel<B>, *reinterpret_cast<const GemmMaps*>(e.host_blob),
                                    (__nv_bfloat16*)e.out, N);
        }
      }
      if constexpr (B >= 192) {  // persistent, TMEM double-buffered (one CTA per SM)
        static const cudaError_t attrp =
            cudaFuncSetAttribute(gemm_persistent_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (attrp != cudaSuccess) return attrp;
        gemm_persistent_kernel<B><<<tiles < sms ? tiles : sms, B, kSmem, s>>>(
            *reinterpret_cast<const GemmMaps*>(e.host_blob), (__nv_bfloat16*)e.out, N);
        return cudaGetLastError();
      }
      gemm_kernel<B><<<tiles, B, kSmem, s>>>(*reinterpret_cast<const GemmMaps*>(e.host_blob),
                                             (__nv_bfloat16*)e.out, N);
      return cudaGetLastError();
    } else {
      return cudaErrorInvalidConfiguration;
    }
  }
};

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

bool make_map(CUtensorMap* m, void* base, int n, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};           // {K, rows}
  cuuint64_t strides[1] = {(cuuint64_t)n * 2};                   // row pitch in bytes
  cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};                // 64 bf16 = 128 B inner
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t gemm_prepare(SuiteEntry& e) {
  static_assert(sizeof(GemmMaps) <= sizeof(e.host_blob), "host blob too small");
  if (e.n % 8 != 0) return cudaErrorInvalidValue;  // TMA row pitch must be 16-byte aligned
  GemmMaps* m = reinterpret_cast<GemmMaps*>(e.host_blob);
  if (!make_map(&m->a, e.in0, (int)e.n, BM) || !make_map(&m->b, e.in1, (int)e.n, BN) ||
      !make_map(&m->b128, e.in1, (int)e.n, 128))
    return cudaErrorInvalidValue;
  return cudaSuccess;
}

const KernelTable& table_gemm() { static KernelTable t = make_table<GemmL>(); return t; }

}  // namespace lscat
