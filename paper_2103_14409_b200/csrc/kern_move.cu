// kern_move.cu — data-movement members of the suite: transpose, axpy, 5-point stencil, and
// the test-only spin kernel.  All HBM bound.
#include "kern_common.cuh"

namespace lscat {
namespace {

// ---------------------------------------------------------------- transpose -------------
// 32x32 tile through padded shared memory (bank-conflict free), threads (32, B/32): each
// thread row moves 32/(B/32) tile rows.  Coalesced 128-byte row segments in and out.
template <int B>
__global__ void __launch_bounds__(B) transpose_kernel(const float* __restrict__ A,
                                                      float* __restrict__ T, int N) {
  constexpr int TY = B / 32;
  __shared__ float tile[32][33];
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const int x = bx + lx;
  if (x < N) {
#pragma unroll
    for (int i = ly; i < 32; i += TY)
      if (by + i < N) tile[i][lx] = ld_stream(A + (size_t)(by + i) * N + x);
  }
  __syncthreads();
  const int x2 = by + lx;
  if (x2 < N) {
#pragma unroll
    for (int i = ly; i < 32; i += TY)
      if (bx + i < N) st_stream(T + (size_t)(bx + i) * N + x2, tile[lx][i]);
  }
}

template <int B>
struct TransposeL {
  static constexpr bool kSupported = true;
  static int occupancy() { return occupancy_warps(transpose_kernel<B>, B); }
  static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
    const SuiteEntry& e = *a.e;
    const int N = (int)e.n;
    dim3 grid((N + 31) / 32, (N + 31) / 32);
    transpose_kernel<B><<<grid, B, 0, s>>>((const float*)e.in0, (float*)e.out, N);
    return cudaGetLastError();
  }
};

// ---------------------------------------------------------------- axpy ------------------
// z = alpha x + y over n = N^2 elements, alpha = 0.5.  Each thread moves U float4 of x and of
// y (2U independent 128-bit loads in flight), streaming loads and stores.
constexpr int kAxpyU = 4;

template <int B>
__global__ void __launch_bounds__(B) axpy_kernel4(const float4* __restrict__ x,
                                                  const float4* __restrict__ y,
                                                  float4* __restrict__ z, size_t n4) {
  const size_t base = (size_t)blockIdx.x * (B * kAxpyU) + threadIdx.x;
  float4 a[kAxpyU], b[kAxpyU];
#pragma unroll
  for (int u = 0; u < kAxpyU; u++) {
    const size_t j = base + (size_t)u * B;
    if (j < n4) { a[u] = ld_stream(x + j); b[u] = ld_stream(y + j); }
  }
#pragma unroll
  for (int u = 0; u < kAxpyU; u++) {
    const size_t j = base + (size_t)u * B;
    if (j < n4) {
      float4 r;
      r.x = fmaf(0.5f, a[u].x, b[u].x); r.y = fmaf(0.5f, a[u].y, b[u].y);
      r.z = fmaf(0.5f, a[u].z, b[u].z); r.w = fmaf(0.5f, a[u].w, b[u].w);
      st_stream(z + j, r);
    }
  }
}

template <int B>
__global__ void __launch_bounds__(B) axpy_kernel1(const float* __restrict__ x,
                                                  const float* __restrict__ y,
                                                  float* __restrict__ z, size_t n) {
  const size_t base = (size_t)blockIdx.x * (B * kAxpyU) + threadIdx.x;
#pragma unroll
  for (int u = 0; u < kAxpyU; u++) {
    const size_t j = base + (size_t)u * B;
    if (j < n) st_stream(z + j, fmaf(0.5f, ld_stream(x + j), ld_stream(y + j)));
  }
}

template <int B>
struct AxpyL {
  static constexpr bool kSupported = true;
  static int occupancy() { return occupancy_warps(axpy_kernel4<B>, B); }
  static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
    const SuiteEntry& e = *a.e;
    const size_t n = (size_t)e.n * e.n;
    if ((n & 3) == 0) {
      const size_t n4 = n / 4;
      const size_t grid = (n4 + (size_t)B * kAxpyU - 1) / ((size_t)B * kAxpyU);
      axpy_kernel4<B><<<(unsigned)grid, B, 0, s>>>((const float4*)e.in0, (const float4*)e.in1,
                                                   (float4*)e.out, n4);
    } else {
      const size_t grid = (n + (size_t)B * kAxpyU - 1) / ((size_t)B * kAxpyU);
      axpy_kernel1<B><<<(unsigned)grid, B, 0, s>>>((const float*)e.in0, (const float*)e.in1,
                                                   (float*)e.out, n);
    }
    return cudaGetLastError();
  }
};

// ---------------------------------------------------------------- stencil5 --------------
// out = c0 A[i][j] + c1 (A[i-1][j] + A[i+1][j] + A[i][j-1] + A[i][j+1]) inside, border copied.
// Threads (32, B/32); a warp owns 32*VEC columns and walks a strip of S rows keeping the rows
// above/at/below in registers (each row loaded once per strip); left/right neighbours come
// from the adjacent lanes by shuffle, the two warp-edge columns by one scalar load each.
constexpr int kStencilS = 8;
constexpr float kC0 = 0.5f, kC1 = 0.125f;

template <int VEC>
struct Vec;
template <>
struct Vec<4> {
  using T = float4;
  static __device__ __forceinline__ T load(const float* p) { return ld_stream(reinterpret_cast<const float4*>(p)); }
  static __device__ __forceinline__ float get(const T& v, int c) { return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w; }
  static __device__ __forceinline__ void set(T& v, int c, float f) { if (c == 0) v.x = f; else if (c == 1) v.y = f; else if (c == 2) v.z = f; else v.w = f; }
  static __device__ __forceinline__ void store(float* p, const T& v) { st_stream(reinterpret_cast<float4*>(p), v); }
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
};
template <>
struct Vec<1> {
  using T = float;
  static __device__ __forceinline__ T load(const float* p) { return ld_stream(p); }
  static __device__ __forceinline__ float get(const T& v, int) { return v; }
  static __device__ __forceinline__ void set(T& v, int, float f) { v = f; }
  static __device__ __forceinline__ void store(float* p, const T& v) { st_stream(p, v); }
  static __device__ __forceinline__ T zero() { return 0.f; }
};

template <int B, int VEC>
__global__ void __launch_bounds__(B) stencil_kernel(const float* __restrict__ A,
                                                    float* __restrict__ out, int N) {
  using V = Vec<VEC>;
  using T = typename V::T;
  constexpr int TY = B / 32;
  const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int col0 = blockIdx.x * (32 * VEC) + lane * VEC;
  const bool valid = col0 < N;
  const int r0 = (blockIdx.y * TY + ty) * kStencilS;
  if (r0 >= N) return;  // whole warp leaves together (r0 is warp-uniform)
  const int r1 = min(r0 + kStencilS, N);
  T up = V::zero(), cur = V::zero(), dn = V::zero();
  if (valid) {
    if (r0 > 0) up = V::load(A + (size_t)(r0 - 1) * N + col0);
    cur = V::load(A + (size_t)r0 * N + col0);
  }
  for (int i = r0; i < r1; i++) {
    if (valid && i + 1 < N) dn = V::load(A + (size_t)(i + 1) * N + col0);
    // neighbours across lanes
    float left = __shfl_up_sync(0xffffffffu, V::get(cur, VEC - 1), 1);
    float right = __shfl_down_sync(0xffffffffu, V::get(cur, 0), 1);
    if (valid) {
      if (lane == 0 && col0 > 0) left = ld_stream(A + (size_t)i * N + col0 - 1);
      if ((lane == 31 || col0 + VEC >= N) && col0 + VEC < N)
        right = ld_stream(A + (size_t)i * N + col0 + VEC);
      T o = cur;
      const bool row_border = (i == 0 || i == N - 1);
#pragma unroll
      for (int c = 0; c < VEC; c++) {
        const int j = col0 + c;
        if (j >= N) break;
        if (row_border || j == 0 || j == N - 1) continue;  // copy
        const float l = c == 0 ? left : V::get(cur, c - 1);
        const float r = c == VEC - 1 ? right : V::get(cur, c + 1);
        const float nb = (V::get(up, c) + V::get(dn, c)) + (l + r);
        V::set(o, c, fmaf(kC0, V::get(cur, c), kC1 * nb));
      }
      if (col0 + VEC <= N) {
        V::store(out + (size_t)i * N + col0, o);
      } else {
        for (int c = 0; c < VEC && col0 + c < N; c++) out[(size_t)i * N + col0 + c] = V::get(o, c);
      }
    }
    up = cur;
    cur = dn;
  }
}

template <int B>
struct StencilL {
  static constexpr bool kSupported = true;
  static int occupancy() { return occupancy_warps(stencil_kernel<B, 4>, B); }
  static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
    const SuiteEntry& e = *a.e;
    const int N = (int)e.n;
    constexpr int TY = B / 32;
    const int rows_per_cta = TY * kStencilS;
    if ((N & 3) == 0) {
      dim3 grid((N + 127) / 128, (N + rows_per_cta - 1) / rows_per_cta);
      stencil_kernel<B, 4><<<grid, B, 0, s>>>((const float*)e.in0, (float*)e.out, N);
    } else {
      dim3 grid((N + 31) / 32, (N + rows_per_cta - 1) / rows_per_cta);
      stencil_kernel<B, 1><<<grid, B, 0, s>>>((const float*)e.in0, (float*)e.out, N);
    }
    return cudaGetLastError();
  }
};

// ---------------------------------------------------------------- spin (tests) ----------
template <int B>
__global__ void __launch_bounds__(B) spin_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

template <int B>
struct SpinL {
  static constexpr bool kSupported = true;
  static int occupancy() { return occupancy_warps(spin_kernel<B>, B); }
  static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
    spin_kernel<B><<<1, B, 0, s>>>(a.spin_ns);
    return cudaGetLastError();
  }
};

}  // namespace

const KernelTable& table_transpose() { static KernelTable t = make_table<TransposeL>(); return t; }
const KernelTable& table_axpy() { static KernelTable t = make_table<AxpyL>(); return t; }
const KernelTable& table_stencil5() { static KernelTable t = make_table<StencilL>(); return t; }
const KernelTable& table_spin() { static KernelTable t = make_table<SpinL>(); return t; }

}  // namespace lscat
