// Probe: where a small-N row-kernel launch spends its ~1.7 us in a plain CUDA graph (the
// empty kernel takes ~0.44 us).  Variants of a one-warp-per-row euclid at N = 64 / 256:
//   0 full (loads of A and q, reduce, store)   1 no store   2 no loads (store a constant)
//   3 loads of A only (q from a constant)      4 full, A via ld.global (default caching)
// Each: a graph of 1000 dependent launches, timed with events, per-launch us printed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lfp scripts/launch_floor_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int B, int V>
__global__ void __launch_bounds__(B) rowk(const float* __restrict__ A, const float* __restrict__ q,
                                         float* __restrict__ out, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * (B / 32) + warp;
  if (row >= N) return;
  float s = 0.f;
  if (V != 2) {
    const float4* a4 = reinterpret_cast<const float4*>(A + (size_t)row * N);
    const float4* q4 = reinterpret_cast<const float4*>(q);
    for (int j = lane; j < N / 4; j += 32) {
      float4 a;
      if (V == 4) a = a4[j];
      else asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(a4 + j));
      const float4 v = V == 3 ? make_float4(0.5f, 0.5f, 0.5f, 0.5f) : __ldg(q4 + j);
      const float d0 = a.x - v.x, d1 = a.y - v.y, d2 = a.z - v.z, d3 = a.w - v.w;
      s += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  } else {
    s = 1.f;
  }
  if (V != 1 && lane == 0) out[row] = sqrtf(s);
}

__global__ void emptyk() {}

template <typename F>
float time_graph(F launch, cudaStream_t s) {
  cudaGraph_t g;
  cudaGraphExec_t gx;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 1000; i++) launch(s);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&gx, g, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaGraphLaunch(gx, s);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 5; r++) cudaGraphLaunch(gx, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / 5000.f;  // us per launch
}

template <int B>
void run(int N, float* A, float* q, float* o, cudaStream_t s) {
  const int grid = (N + B / 32 - 1) / (B / 32);
  printf("N=%d B=%d: full %.3f  nostore %.3f  noload %.3f  Aonly %.3f  cachedA %.3f us\n", N, B,
         time_graph([&](cudaStream_t t) { rowk<B, 0><<<grid, B, 0, t>>>(A, q, o, N); }, s),
         time_graph([&](cudaStream_t t) { rowk<B, 1><<<grid, B, 0, t>>>(A, q, o, N); }, s),
         time_graph([&](cudaStream_t t) { rowk<B, 2><<<grid, B, 0, t>>>(A, q, o, N); }, s),
         time_graph([&](cudaStream_t t) { rowk<B, 3><<<grid, B, 0, t>>>(A, q, o, N); }, s),
         time_graph([&](cudaStream_t t) { rowk<B, 4><<<grid, B, 0, t>>>(A, q, o, N); }, s));
}

int main() {
  float *A, *q, *o;
  cudaMalloc(&A, 4096 * 4096 * 4);
  cudaMalloc(&q, 4096 * 4);
  cudaMalloc(&o, 4096 * 4);
  cudaMemset(A, 0, 4096 * 4096 * 4);
  cudaMemset(q, 0, 4096 * 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  printf("empty kernel (1 x 32): %.3f us\n", time_graph([&](cudaStream_t t) { emptyk<<<1, 32, 0, t>>>(); }, s));
  printf("empty kernel (64 x 32): %.3f us\n", time_graph([&](cudaStream_t t) { emptyk<<<64, 32, 0, t>>>(); }, s));
  printf("empty kernel (2 x 1024): %.3f us\n", time_graph([&](cudaStream_t t) { emptyk<<<2, 1024, 0, t>>>(); }, s));
  for (int N : {64, 256, 1024}) {
    run<32>(N, A, q, o, s);
    run<256>(N, A, q, o, s);
    run<1024>(N, A, q, o, s);
  }
  return 0;
}
