// kern_cols.cu — column reduction c[j] = sum_i A[i][j] (suite member).
//
// Mapping: a CTA owns a column tile (128 columns: 32 lanes x float4; 32 columns on the scalar
// path for N % 4 != 0) and a chunk of rows; its B/32 warps stride over the chunk's rows with
// U independent 128-bit loads in flight.  Warps are combined in smem in a fixed order, chunk
// partials go to scratch, and the last CTA of a tile (atomic ticket) sums the chunks in chunk
// order: a single launch, deterministic (no floating-point atomics).  HBM: 4N^2 + 4N bytes.
#include "kern_common.cuh"

namespace lscat {
namespace {

constexpr int kMaxChunks = 64;

inline int colsum_chunks(int N, int B) {
  const int W = B / 32;
  int c = (N + W * 16 - 1) / (W * 16);  // >= 16 rows per warp
  return c < 1 ? 1 : (c > kMaxChunks ? kMaxChunks : c);
}

template <int B, int VEC>
__global__ void __launch_bounds__(B, min_blocks_64regs<B>()) colsum_kernel(const float* __restrict__ A,
                                                   float* __restrict__ out,
                                                   float* __restrict__ partials,
                                                   unsigned* __restrict__ tickets, int N,
                                                   int chunks, int rows_per_chunk) {
  constexpr int W = B / 32;
  constexpr int TC = 32 * VEC;  // columns per tile
  __shared__ float red[W][TC];
  __shared__ unsigned is_last;
  pdl_trigger();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int col = blockIdx.x * TC + lane * VEC;
  const int r0 = blockIdx.y * rows_per_chunk;
  const int r1 = min(r0 + rows_per_chunk, N);
  float acc[VEC];
#pragma unroll
  for (int c = 0; c < VEC; c++) acc[c] = 0.f;
  if (col < N) {
    constexpr int U = 4;
    for (int r = r0 + w; r < r1; r += U * W) {
      if constexpr (VEC == 4) {
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int rr = r + u * W;
          x[u] = rr < r1 ? ld_stream(reinterpret_cast<const float4*>(A + (size_t)rr * N + col))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          acc[0] += x[u].x; acc[1] += x[u].y; acc[2] += x[u].z; acc[3] += x[u].w;
        }
      } else {
        float x[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int rr = r + u * W;
          x[u] = rr < r1 ? ld_stream(A + (size_t)rr * N + col) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; u++) acc[0] += x[u];
      }
    }
  }
  pdl_wait();  // partials / tickets / out are shared with the previous launch
#pragma unroll
  for (int c = 0; c < VEC; c++) red[w][lane * VEC + c] = acc[c];
  __syncthreads();
  // fixed-order combine of the W warps; thread t handles tile columns t, t+B, ...
  for (int tc = threadIdx.x; tc < TC; tc += B) {
    float s = 0.f;
#pragma unroll 8
    for (int k = 0; k < W; k++) s += red[k][tc];
    const int j = blockIdx.x * TC + tc;
    if (j < N) {
      if (chunks == 1) out[j] = s;
      else partials[(size_t)blockIdx.y * N + j] = s;
    }
  }
  if (chunks == 1) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(&tickets[blockIdx.x], 1u) == (unsigned)chunks - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int tc = threadIdx.x; tc < TC; tc += B) {
    const int j = blockIdx.x * TC + tc;
    if (j >= N) continue;
    float s = 0.f;
#pragma unroll 16
    for (int k = 0; k < chunks; k++) s += __ldcg(partials + (size_t)k * N + j);
    out[j] = s;
  }
  if (threadIdx.x == 0) tickets[blockIdx.x] = 0;  // re-arm for the next launch
}

template <int B>
struct ColsumL {
  static constexpr bool kSupported = true;
  static cudaError_t attrs(const void** f, size_t* sm) { return kernel_attrs(colsum_kernel<B, 4>, 0, f, sm); }
  static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
    const SuiteEntry& e = *a.e;
    const int N = (int)e.n;
    const int chunks = colsum_chunks(N, B);
    const int rpc = (N + chunks - 1) / chunks;
    float* partials = (float*)e.scratch;
    unsigned* tickets = (unsigned*)((char*)e.scratch + (size_t)kMaxChunks * N * sizeof(float));
    if ((N & 3) == 0) {
      dim3 grid((N + 127) / 128, chunks);
      return launch_k(colsum_kernel<B, 4>, grid, dim3(B), 0, s, a.pdl, (const float*)e.in0, (float*)e.out,
                      partials, tickets, N, chunks, rpc);
    } else {
      dim3 grid((N + 31) / 32, chunks);
      return launch_k(colsum_kernel<B, 1>, grid, dim3(B), 0, s, a.pdl, (const float*)e.in0, (float*)e.out,
                      partials, tickets, N, chunks, rpc);
    }
  }
};

}  // namespace

cudaError_t colsum_prepare(SuiteEntry& e) {
  const size_t N = e.n;
  e.scratch_bytes = (size_t)kMaxChunks * N * sizeof(float) + ((N + 31) / 32) * sizeof(unsigned);
  cudaError_t err = cudaMalloc(&e.scratch, e.scratch_bytes);
  if (err != cudaSuccess) return err;
  return cudaMemset(e.scratch, 0, e.scratch_bytes);
}

const KernelTable& table_colsum() { static KernelTable t = make_table<ColsumL>(); return t; }

}  // namespace lscat
