// Probe 2: which part of the library's row kernel (kern_rows.cu) costs the extra ~0.5-1.3 us per
// small-N launch against a bare one-warp-per-row kernel.  Feature bits of variant F:
//   1 griddepcontrol.launch_dependents at entry + griddepcontrol.wait before the store (PDL)
//   2 fractional L2 evict-last policy on A's loads (createpolicy + cache_hint)
//   4 8 predicated float4 loads per lane per pass (U = 8), like the library
//   8 a static shared array + the team-combine branch structure
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int B, int F>
__global__ void __launch_bounds__(B, (1024 / B) > 0 ? 1024 / B : 1) rowk(const float* __restrict__ A,
                                                                          const float* __restrict__ q,
                                                                          float* __restrict__ out, int N) {
  __shared__ float red[B / 32];
  if (F & 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * (B / 32) + warp;
  float s = 0.f;
  uint64_t pol = 0;
  if (F & 2) asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(pol) : "f"(1.0f));
  if (row < N) {
    const float4* a4 = reinterpret_cast<const float4*>(A + (size_t)row * N);
    const float4* q4 = reinterpret_cast<const float4*>(q);
    const int n4 = N / 4;
    constexpr int U = (F & 4) ? 8 : 1;
    for (int base = lane; base < n4; base += U * 32) {
      float4 x[U], y[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int j = base + u * 32;
        if (j < n4) {
          if (F & 2)
            asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                : "=f"(x[u].x), "=f"(x[u].y), "=f"(x[u].z), "=f"(x[u].w) : "l"(a4 + j), "l"(pol));
          else
            asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(x[u].x), "=f"(x[u].y), "=f"(x[u].z), "=f"(x[u].w) : "l"(a4 + j));
          y[u] = __ldg(q4 + j);
        } else {
          x[u] = y[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const float d0 = x[u].x - y[u].x, d1 = x[u].y - y[u].y, d2 = x[u].z - y[u].z, d3 = x[u].w - y[u].w;
        s += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (F & 8) {
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (lane == 0) s = red[warp];
    __syncthreads();
  }
  if (F & 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (row < N && lane == 0) out[row] = sqrtf(s);
}

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
  return ms * 1000.f / 5000.f;
}

template <int B, int F>
float one(int N, float* A, float* q, float* o, cudaStream_t s) {
  const int grid = (N + B / 32 - 1) / (B / 32);
  return time_graph([&](cudaStream_t t) { rowk<B, F><<<grid, B, 0, t>>>(A, q, o, N); }, s);
}

template <int B>
void run(int N, float* A, float* q, float* o, cudaStream_t s) {
  printf("N=%d B=%d: base %.3f pdl %.3f pol %.3f u8 %.3f smem %.3f all %.3f all-but-u8 %.3f us\n", N, B,
         one<B, 0>(N, A, q, o, s), one<B, 1>(N, A, q, o, s), one<B, 2>(N, A, q, o, s),
         one<B, 4>(N, A, q, o, s), one<B, 8>(N, A, q, o, s), one<B, 15>(N, A, q, o, s),
         one<B, 11>(N, A, q, o, s));
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
  for (int N : {64, 256, 1024, 2048, 4096}) {
    run<32>(N, A, q, o, s);
    run<128>(N, A, q, o, s);
    run<256>(N, A, q, o, s);
    run<512>(N, A, q, o, s);
    run<1024>(N, A, q, o, s);
  }
  return 0;
}
