// kern_common.cuh — device helpers shared by the suite kernels (not by the reducer).
#pragma once
#include <cuda_runtime.h>

#include <utility>

#include "common.h"

namespace lscat {

// Streaming 128-bit load: read-only path, no L1 allocation (each element is read once).
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
// Same load with an L2 evict-last cache policy (from createpolicy): for inputs that fit in L2
// and are re-read by the next launch.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Fractional policy: a fixed (address-hashed) fraction of the lines accessed is kept with
// evict-last priority, the rest streams through with evict-first, so a buffer larger than L2
// leaves a stable resident part instead of thrashing.
__device__ __forceinline__ uint64_t l2_keep_fraction_policy(float frac) {
  uint64_t pol;
#ifdef L2_SECONDARY_UNCHANGED
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, %1;" : "=l"(pol) : "f"(frac));
#else
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(pol) : "f"(frac));
#endif
  return pol;
}
__device__ __forceinline__ float4 ld_keep(const float4* p, uint64_t pol) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(p), "l"(pol));
  return r;
}
// Streaming store (evict-first in L2, the output is not re-read by this launch).
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }

// Minimum resident CTAs declared in __launch_bounds__ so that ptxas budgets 64 registers per
// thread (32 warps per SM).  Without it ptxas sizes registers for full occupancy (32 per
// thread for B >= 64) and serialises independent 128-bit loads (one in flight per thread).
template <int B>
constexpr int min_blocks_64regs() { return 1024 / B > 0 ? 1024 / B : 1; }

// Programmatic dependent launch (PDL).  A suite kernel triggers its dependents at entry and
// waits for its predecessor grid (completion + memory flush) before its first global store,
// so in a back-to-back bracket launch i+1's CTAs are scheduled, and issue their loads of the
// read-only inputs, while launch i drains.  Both are no-ops for a launch without the
// programmatic-serialisation attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            bool pdl, Args... args) {
  if (!pdl) {
    k<<<grid, block, smem, s>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

template <int B>
__device__ __forceinline__ float block_sum(float v, float* red /* [B/32] smem */) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if constexpr (B == 32) {
    return v;
  } else {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = v;
    __syncthreads();
    v = (l < B / 32) ? red[l] : 0.f;
    if (w == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;  // valid in warp 0
  }
}

// The device function of a launch and its dynamic shared memory (AttrFn in common.h).
template <typename F>
inline cudaError_t kernel_attrs(F kernel, size_t dyn, const void** f, size_t* smem) {
  *f = (const void*)kernel;
  *smem = dyn;
  if (dyn > 48 * 1024)
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  return cudaSuccess;
}

// Builds a KernelTable whose entry i launches Launcher<32*(i+1)>::launch (or nullptr when
// Launcher<B>::kSupported is false).
template <template <int> class Launcher, int... Is>
KernelTable make_table_impl(std::integer_sequence<int, Is...>) {
  KernelTable t{};
  ((t.fn[Is] = Launcher<32 * (Is + 1)>::kSupported ? &Launcher<32 * (Is + 1)>::launch : nullptr),
   ...);
  ((t.attrs[Is] = Launcher<32 * (Is + 1)>::kSupported ? &Launcher<32 * (Is + 1)>::attrs : nullptr),
   ...);
  return t;
}
template <template <int> class Launcher>
KernelTable make_table() {
  return make_table_impl<Launcher>(std::make_integer_sequence<int, kMaxBlockIdx>{});
}

}  // namespace lscat
