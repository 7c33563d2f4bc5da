// Minimal reproducer for the racecheck reports on the CTA-pair GEMM (profiles/r02_racecheck.txt):
// the allocator pattern of gemm_2cta_kernel and nothing else.  One warp per CTA of a 2-CTA
// cluster issues tcgen05.alloc.cta_group::2 into a shared-memory slot, relinquishes the permit,
// both CTAs cross a cluster barrier (release/acquire) and every thread reads the slot, then one
// warp deallocates after a second cluster barrier.  The cta_group::1 variant does the same per
// CTA with a CTA barrier.  If racecheck reports hazards on the pair variant of this program, the
// reports on the GEMM are the tool's model of the pair-collective allocation, not a race in it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/rc scripts/racecheck_tmem_pair.cu
//   compute-sanitizer --tool racecheck /tmp/rc 2 ; compute-sanitizer --tool racecheck /tmp/rc 1
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__global__ void __cluster_dims__(2, 1, 1) pair_alloc(unsigned* out) {
  __shared__ unsigned slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = tmem;
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

__global__ void single_alloc(unsigned* out) {
  __shared__ unsigned slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = tmem;
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 2;
  unsigned* d = nullptr;
  cudaMalloc(&d, 8 * sizeof(unsigned));
  if (mode == 2) pair_alloc<<<2, 128>>>(d);
  else single_alloc<<<2, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned h[2] = {0, 0};
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("mode %d: %s, tmem addresses %u %u\n", mode, cudaGetErrorString(e), h[0], h[1]);
  return e == cudaSuccess ? 0 : 1;
}
