// Transpose calibration (round 2): standalone probe of band-shaped CTA tiles for the N x N fp32
// transpose.  The library kernel (per-warp 64 x 32 units: 128 B read runs, 256 B write runs) is
// compared with CTA tiles of R rows x C columns that read long row runs (C * 4 B) and write
// R * 4 B runs (32-128 B: whole sectors, merged into lines in L2 by the neighbouring bands that
// run concurrently).  Cold L2: a 512 MB memset before every timed launch.  Prints one line per
// variant: median / min us over the reps and GB/s at 8 N^2 bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tpb scripts/tp_band_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// ---- the library's kernel (TP_TPW 2, vertical) -------------------------------------------
template <int B>
__global__ void __launch_bounds__(B, (768 / B) > 0 ? 768 / B : 1) tp_lib(const float* __restrict__ A, float* __restrict__ T, int N, int units_x, int nunits) {
  constexpr int W = B / 32, U = 2;
  extern __shared__ float tp_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float(*t)[33] = reinterpret_cast<float(*)[33]>(tp_smem + w * (32 * 33));
  const int r = lane >> 3, c = (lane & 7) * 4;
  for (int id = blockIdx.x * W + w; id < nunits; id += gridDim.x * W) {
    const int by0 = (id / units_x) * 64, bx0 = (id % units_x) * 32;
    float4 v[U][8];
#pragma unroll
    for (int u = 0; u < U; u++)
#pragma unroll
      for (int i = 0; i < 8; i++) v[u][i] = ld_stream(reinterpret_cast<const float4*>(A + (size_t)(by0 + 32 * u + r + 4 * i) * N + bx0 + c));
#pragma unroll
    for (int u = 0; u < U; u++) {
#pragma unroll
      for (int i = 0; i < 8; i++) {
        t[r + 4 * i][c + 0] = v[u][i].x; t[r + 4 * i][c + 1] = v[u][i].y;
        t[r + 4 * i][c + 2] = v[u][i].z; t[r + 4 * i][c + 3] = v[u][i].w;
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int o = r + 4 * i;
        const float4 q = make_float4(t[c + 0][o], t[c + 1][o], t[c + 2][o], t[c + 3][o]);
        __stcs(reinterpret_cast<float4*>(T + (size_t)(bx0 + o) * N + by0 + 32 * u + c), q);
      }
      __syncwarp();
    }
  }
}

// ---- band tiles: R rows x C cols per CTA tile, B threads, persistent grid --------------
// load: float4 per thread along rows, all R*C/(4B) float4 of the tile in flight per thread;
// smem [R][C] with the 16 B chunks of row r XOR-swizzled by f(r) = ((r / 4) * max(1, 8 / L)) % 8
// (the L lanes of an output row read rows 4j..4j+3 at the same column: distinct banks); store: L = R/4 lanes per output row, each writes one float4 of
// rows 4j..4j+3 -> a warp instruction covers 32/L output rows of R*4 B.
// ORDER 0: tile id row-major (bands of R rows, C-column blocks); 1: column-major.
template <int B, int R, int C, int ORDER>
__global__ void __launch_bounds__(B) tp_band(const float* __restrict__ A, float* __restrict__ T, int N) {
  constexpr int L = R / 4, CP = C, SWM = (8 / L) > 0 ? 8 / L : 1, NV = R * C / 4 / B, RPW = 32 / L;  // rows per warp instr
  static_assert(NV >= 1, "tile too small for the block");
  extern __shared__ float sm[];
  const int tiles_x = N / C, tiles_y = N / R, ntiles = tiles_x * tiles_y;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int ty = ORDER == 0 ? t / tiles_x : t % tiles_y, tx = ORDER == 0 ? t % tiles_x : t / tiles_y;
    const int y0 = ty * R, x0 = tx * C;
    float4 v[NV];
#pragma unroll
    for (int k = 0; k < NV; k++) {
      const int e = (k * B + tid) * 4, rr = e / C, cc = e % C;
      v[k] = ld_stream(reinterpret_cast<const float4*>(A + (size_t)(y0 + rr) * N + x0 + cc));
    }
    __syncthreads();  // previous tile's smem reads done
#pragma unroll
    for (int k = 0; k < NV; k++) {
      const int e = (k * B + tid) * 4, rr = e / C, cc = e % C;
      *reinterpret_cast<float4*>(&sm[rr * CP + (cc ^ ((((rr >> 2) * SWM) & 7) << 2))]) = v[k];
    }
    __syncthreads();
    // store: warp w handles output rows (input cols) in chunks of RPW
    const int j = lane % L, xr = lane / L;
    for (int xb = w * RPW; xb < C; xb += (B / 32) * RPW) {
      const int x = xb + xr;
      const int xs = x ^ (((j * SWM) & 7) << 2);  // rows 4j..4j+3 share the swizzle
      const float4 q = make_float4(sm[(4 * j + 0) * CP + xs], sm[(4 * j + 1) * CP + xs], sm[(4 * j + 2) * CP + xs],
                                   sm[(4 * j + 3) * CP + xs]);
      __stcs(reinterpret_cast<float4*>(T + (size_t)(x0 + x) * N + y0 + 4 * j), q);
    }
  }
}

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) __stcs(b + i, ld_stream(a + i));
}

__global__ void fill_k(float* a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    a[i] = (float)((i * 2654435761u) % 1000003) * 1e-3f;
}

__global__ void check_k(const float* A, const float* T, int N, unsigned long long* bad) {
  size_t n = (size_t)N * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    size_t r = i / N, c = i % N;
    if (T[c * N + r] != A[i]) atomicAdd(bad, 1ull);
  }
}

static int N = 8192, REPS = 15, SMS = 148;
static float *dA, *dT, *dF;
static unsigned long long* dBad;
static size_t flushB = 512ull << 20;

template <typename F>
static void run(const char* name, F launch, bool check = true) {
  std::vector<float> ts;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaMemset(dT, 0, (size_t)N * N * 4));
  launch();
  CK(cudaDeviceSynchronize());
  if (check) {
    CK(cudaMemset(dBad, 0, 8));
    check_k<<<SMS * 8, 256>>>(dA, dT, N, dBad);
    unsigned long long bad = 0;
    CK(cudaMemcpy(&bad, dBad, 8, cudaMemcpyDeviceToHost));
    if (bad) { printf("%-28s WRONG (%llu)\n", name, bad); return; }
  }
  for (int r = 0; r < REPS; r++) {
    CK(cudaMemsetAsync(dF, r, flushB));
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    ts.push_back(ms * 1e3f);
  }
  CK(cudaGetLastError());
  std::sort(ts.begin(), ts.end());
  const double bytes = 8.0 * N * N;
  printf("%-28s med %7.1f us  min %7.1f us  %6.0f GB/s (med)\n", name, ts[ts.size() / 2], ts[0], bytes / (ts[ts.size() / 2] * 1e3));
}

template <int B, int R, int C, int ORDER>
static void band(int per_sm_override = 0) {
  constexpr int smem = R * C * 4;
  auto k = tp_band<B, R, C, ORDER>;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, B, smem));
  if (per_sm_override) per = std::min(per, per_sm_override);
  const int ntiles = (N / C) * (N / R), grid = std::min(ntiles, per * SMS);
  char name[96];
  snprintf(name, sizeof name, "band B%d R%d C%d o%d x%d", B, R, C, ORDER, per);
  run(name, [=] { k<<<grid, B, smem>>>(dA, dT, N); });
}

template <int B>
static void lib() {
  constexpr int smem = (B / 32) * 32 * 33 * 4;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(tp_lib<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tp_lib<B>, B, smem));
  const int units_x = N / 32, nunits = units_x * (N / 64), need = nunits / (B / 32);
  const int grid = std::min(need, per * SMS);
  char name[64];
  snprintf(name, sizeof name, "lib B%d x%d", B, per);
  run(name, [=] { tp_lib<B><<<grid, B, smem>>>(dA, dT, N, units_x, nunits); });
}

int main(int argc, char** argv) {
  if (argc > 1) N = atoi(argv[1]);
  CK(cudaDeviceGetAttribute(&SMS, cudaDevAttrMultiProcessorCount, 0));
  const size_t n = (size_t)N * N;
  CK(cudaMalloc(&dA, n * 4)); CK(cudaMalloc(&dT, n * 4)); CK(cudaMalloc(&dF, flushB)); CK(cudaMalloc(&dBad, 8));
  fill_k<<<SMS * 8, 256>>>(dA, n);
  CK(cudaDeviceSynchronize());
  printf("N = %d, SMs %d, cold L2 (512 MB memset before each rep), %d reps\n", N, SMS, REPS);
  run("copy float4 (ceiling)", [=] { copy_k<<<SMS * 8, 512>>>((const float4*)dA, (float4*)dT, n / 4); }, false);
  run("cudaMemcpy D2D", [=] { cudaMemcpyAsync(dT, dA, n * 4, cudaMemcpyDeviceToDevice); }, false);
  lib<256>(); lib<512>(); lib<128>();
  band<256, 8, 1024, 0>(); band<256, 8, 512, 0>(); band<512, 8, 1024, 0>();
  band<256, 16, 512, 0>(); band<256, 16, 1024, 0>(); band<512, 16, 1024, 0>();
  band<256, 32, 256, 0>(); band<256, 32, 512, 0>(); band<512, 32, 512, 0>(); band<512, 32, 1024, 0>();
  band<256, 8, 1024, 1>(); band<256, 16, 512, 1>(); band<256, 32, 256, 1>();
  band<128, 8, 512, 0>(); band<128, 16, 256, 0>(); band<128, 32, 128, 0>();
  band<256, 64, 128, 0>(); band<256, 64, 256, 0>(); band<256, 128, 128, 0>();
  return 0;
}
