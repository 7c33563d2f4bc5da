// grid.sync() cost on B200: 148 CTAs x {1024, 256} threads, 200 barriers per launch, events.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gs scripts/gridsync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; i++) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

// sense-reversing barrier on one global word (thread 0 per CTA), acquire/release
__global__ void k_own(int iters, unsigned* bar, unsigned* sink) {
  unsigned gen = 0;
  for (int i = 0; i < iters; i++) {
    __syncthreads();
    if (threadIdx.x == 0) {
      gen += gridDim.x;
      __threadfence();
      atomicAdd(bar, 1u);
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar));
      } while (v < gen);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *sink, *bar;
  cudaMalloc(&sink, 64);
  cudaMalloc(&bar, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {1024, 256}) {
    for (int iters : {1, 200}) {
      void* args[] = {(void*)&iters, (void*)&sink};
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((const void*)k_cg, dim3(sms), dim3(threads), args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 2) printf("cg   threads %4d iters %3d: %.1f us total, %.2f us per sync\n", threads, iters, ms * 1e3, ms * 1e3 / iters);
      }
      for (int rep = 0; rep < 3; rep++) {
        cudaMemset(bar, 0, 4);
        void* args2[] = {(void*)&iters, (void*)&bar, (void*)&sink};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((const void*)k_own, dim3(sms), dim3(threads), args2, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 2) printf("own  threads %4d iters %3d: %.1f us total, %.2f us per sync\n", threads, iters, ms * 1e3, ms * 1e3 / iters);
      }
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
