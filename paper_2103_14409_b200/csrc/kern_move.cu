// kern_move.cu — data-movement members of the suite: transpose, axpy, 5-point stencil, and
// the test-only spin kernel.  All HBM bound.
#include "kern_common.cuh"

namespace lscat {
namespace {

// ---------------------------------------------------------------- transpose -------------
// Each WARP transposes units of TP_TPW 32x32 tiles (stacked vertically by default, so an
// output row segment is 32 * TP_TPW contiguous floats) through its own padded smem slice
// (32 x 33 floats); a warp's work does not depend on the block size B (B only groups warps
// into CTAs):
//   load: lane (r = l/8, c = 4(l%8)) reads 8 float4 per tile (rows r, r+4, ..., r+28), all
//         tiles of the unit at once -> 4 KB x TP_TPW of loads in flight per warp; then per tile
//         scalar stores into the slice (bank = r + c + k: conflict-free);
//   store: lane writes output rows r + 4i, columns c..c+3 as one float4 gathered from
//         slice[c..c+3][r + 4i] (bank = c + k + r + 4i: conflict-free), 128 B per output row.
// Persistent grid (occupancy x SMs), warps stride over the units; edge units (or N % 4 != 0)
// take a scalar path.  Only __syncwarp: no CTA barrier.
// B200 calibration (scripts/tp_variants.sh, N = 8192, mean over the 32 blocks): one tile per
// unit 106.9 us; two horizontal 106.5; two vertical 103.8 (this default); four vertical 114.
#ifndef TP_TPW
#define TP_TPW 2  // 32x32 tiles per warp unit (horizontally adjacent): 8 * TP_TPW loads in flight
#endif
#ifndef TP_VERT
#define TP_VERT 1  // 1: the unit's tiles are stacked vertically (longer output row segments)
#endif
#ifndef TP_MINB_THREADS
#define TP_MINB_THREADS 768  // register budget 65536 / TP_MINB_THREADS per thread
#endif
template <int B>
constexpr int tp_min_blocks() { return TP_MINB_THREADS / B > 0 ? TP_MINB_THREADS / B : 1; }

template <int B>
__global__ void __launch_bounds__(B, tp_min_blocks<B>()) transpose_kernel(const float* __restrict__ A,
                                                                         float* __restrict__ T, int N,
                                                                         int units_x, int nunits) {
  constexpr int W = B / 32, U = TP_TPW;
  extern __shared__ float tp_smem[];
  pdl_trigger();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float(*t)[33] = reinterpret_cast<float(*)[33]>(tp_smem + w * (32 * 33));
  const bool vec = (N & 3) == 0;
  const int r = lane >> 3, c = (lane & 7) * 4;
  constexpr int UX = TP_VERT ? 1 : U, UY = TP_VERT ? U : 1;  // unit = UY x UX tiles
  for (int id = blockIdx.x * W + w; id < nunits; id += gridDim.x * W) {
    const int by0 = (id / units_x) * (32 * UY), bx0 = (id % units_x) * (32 * UX);
    if (vec && by0 + 32 * UY <= N && bx0 + 32 * UX <= N) {
      float4 v[U][8];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int by = by0 + (TP_VERT ? 32 * u : 0), bx = bx0 + (TP_VERT ? 0 : 32 * u);
#pragma unroll
        for (int i = 0; i < 8; i++)
          v[u][i] = ld_stream(reinterpret_cast<const float4*>(A + (size_t)(by + r + 4 * i) * N + bx + c));
      }
      pdl_wait();
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int by = by0 + (TP_VERT ? 32 * u : 0), bx = bx0 + (TP_VERT ? 0 : 32 * u);
#pragma unroll
        for (int i = 0; i < 8; i++) {
          t[r + 4 * i][c + 0] = v[u][i].x; t[r + 4 * i][c + 1] = v[u][i].y;
          t[r + 4 * i][c + 2] = v[u][i].z; t[r + 4 * i][c + 3] = v[u][i].w;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const int o = r + 4 * i;  // output row bx + o = input column bx + o
          const float4 q = make_float4(t[c + 0][o], t[c + 1][o], t[c + 2][o], t[c + 3][o]);
          st_stream(reinterpret_cast<float4*>(T + (size_t)(bx + o) * N + by + c), q);
        }
        __syncwarp();  // the slice is rewritten by the next tile
      }
    } else {
      pdl_wait();
      for (int u = 0; u < U; u++) {
        const int by = by0 + (TP_VERT ? 32 * u : 0), bx = bx0 + (TP_VERT ? 0 : 32 * u);
        if (bx >= N || by >= N) break;
        for (int rr = 0; rr < 32; rr++)
          if (by + rr < N && bx + lane < N) t[rr][lane] = ld_stream(A + (size_t)(by + rr) * N + bx + lane);
        __syncwarp();
        for (int cc = 0; cc < 32; cc++)
          if (bx + cc < N && by + lane < N) st_stream(T + (size_t)(bx + cc) * N + by + lane, t[lane][cc]);
        __syncwarp();
      }
    }
  }
}

template <int B>
struct TransposeL {
  static constexpr bool kSupported = true;
  static constexpr int kSmem = (B / 32) * 32 * 33 * (int)sizeof(float);
  // resident CTAs per SM (a property of the sm_100a binary, the same on every device of the
  // process; thread-safe one-time initialisation)
  static int per_sm() {
    static const int v = [] {
      int r = 0;
      if (kSmem > 48 * 1024)
        cudaFuncSetAttribute(transpose_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, transpose_kernel<B>, B, kSmem);
      cudaGetLastError();
      return r > 0 ? r : 1;
    }();
    return v;
  }
  static int grid_cap(int sms) { return (sms > 0 ? sms : 148) * per_sm(); }
  static cudaError_t attrs(const void** f, size_t* sm) { return kernel_attrs(transpose_kernel<B>, kSmem, f, sm); }
  static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
    const SuiteEntry& e = *a.e;
    const int N = (int)e.n;
    constexpr int UX = TP_VERT ? 1 : TP_TPW, UY = TP_VERT ? TP_TPW : 1;
    const int units_x = (N + 32 * UX - 1) / (32 * UX), nunits = units_x * ((N + 32 * UY - 1) / (32 * UY));
    const int need = (nunits + B / 32 - 1) / (B / 32);
    const int cap = grid_cap(a.sms);
    const int grid = need < cap ? need : cap;
    return launch_k(transpose_kernel<B>, dim3(grid), dim3(B), (size_t)kSmem, s, a.pdl, (const float*)e.in0,
                    (float*)e.out, N, units_x, nunits);
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
  pdl_trigger();
  const size_t base = (size_t)blockIdx.x * (B * kAxpyU) + threadIdx.x;
  float4 a[kAxpyU], b[kAxpyU];
#pragma unroll
  for (int u = 0; u < kAxpyU; u++) {
    const size_t j = base + (size_t)u * B;
    if (j < n4) { a[u] = ld_stream(x + j); b[u] = ld_stream(y + j); }
  }
  pdl_wait();
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
  pdl_trigger();
  pdl_wait();
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
  static cudaError_t attrs(const void** f, size_t* sm) { return kernel_attrs(axpy_kernel4<B>, 0, f, sm); }
  static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
    const SuiteEntry& e = *a.e;
    const size_t n = (size_t)e.n * e.n;
    if ((n & 3) == 0) {
      const size_t n4 = n / 4;
      const size_t grid = (n4 + (size_t)B * kAxpyU - 1) / ((size_t)B * kAxpyU);
      return launch_k(axpy_kernel4<B>, dim3((unsigned)grid), dim3(B), 0, s, a.pdl, (const float4*)e.in0,
                      (const float4*)e.in1, (float4*)e.out, n4);
    } else {
      const size_t grid = (n + (size_t)B * kAxpyU - 1) / ((size_t)B * kAxpyU);
      return launch_k(axpy_kernel1<B>, dim3((unsigned)grid), dim3(B), 0, s, a.pdl, (const float*)e.in0,
                      (const float*)e.in1, (float*)e.out, n);
    }
  }
};

// ---------------------------------------------------------------- stencil5 --------------
// out = c0 A[i][j] + c1 (A[i-1][j] + A[i+1][j] + A[i][j-1] + A[i][j+1]) inside, border copied.
// A warp owns 32*VEC columns and a strip of S rows: it loads the S + 2
// rows it needs (strip + halo; the halo rows are L2 hits, shared with the neighbouring
// strips) into registers up front, then computes; left/right neighbours come from the
// adjacent lanes by shuffle, the two warp-edge columns by one scalar load per row.
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
__global__ void __launch_bounds__(B, min_blocks_64regs<B>()) stencil_kernel(const float* __restrict__ A,
                                                                          float* __restrict__ out, int N,
                                                                          int colblocks) {
  using V = Vec<VEC>;
  using T = typename V::T;
  constexpr int S = kStencilS;
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  // global warp -> (strip, column block), column block fastest: concurrent warps cover whole
  // row bands whatever B is.  One strip per warp (a persistent grid-stride version measured
  // slower on B200: 110 vs 83 us at N = 8192, B = 32).
  const int item = blockIdx.x * (B / 32) + (threadIdx.x >> 5);
  {
    const int cb = item % colblocks, strip = item / colblocks;
    const int col0 = cb * (32 * VEC) + lane * VEC;
    const bool valid = col0 < N;
    const int r0 = strip * S;
    if (r0 >= N) return;  // warp-uniform
    // all S + 2 rows of the strip (and the S warp-edge scalars) are loaded before any use:
    // S + 2 independent 128-bit loads in flight per lane
    T rows[S + 2];
#pragma unroll
    for (int k = 0; k < S + 2; k++) {
      const int i = r0 - 1 + k;
      rows[k] = (valid && i >= 0 && i < N) ? V::load(A + (size_t)i * N + col0) : V::zero();
    }
    const bool need_l = valid && lane == 0 && col0 > 0;
    const bool need_r = valid && lane == 31 && col0 + VEC < N;
    const int edge_col = need_l ? col0 - 1 : col0 + VEC;
    float edge[S];
#pragma unroll
    for (int k = 0; k < S; k++)
      edge[k] = ((need_l || need_r) && r0 + k < N) ? ld_stream(A + (size_t)(r0 + k) * N + edge_col) : 0.f;
    pdl_wait();
#pragma unroll
    for (int k = 0; k < S; k++) {
      const int i = r0 + k;
      if (i >= N) break;  // warp-uniform
      const T& up = rows[k];
      const T& cur = rows[k + 1];
      const T& dn = rows[k + 2];
      float left = __shfl_up_sync(0xffffffffu, V::get(cur, VEC - 1), 1);
      float right = __shfl_down_sync(0xffffffffu, V::get(cur, 0), 1);
      if (need_l) left = edge[k];
      if (need_r) right = edge[k];
      if (valid) {
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
    }
  }
}

template <int B>
struct StencilL {
  static constexpr bool kSupported = true;
  static cudaError_t attrs(const void** f, size_t* sm) { return kernel_attrs(stencil_kernel<B, 4>, 0, f, sm); }
  static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
    const SuiteEntry& e = *a.e;
    const int N = (int)e.n;
    const int strips = (N + kStencilS - 1) / kStencilS;
    const int cbs = (N & 3) == 0 ? (N + 127) / 128 : (N + 31) / 32;
    const unsigned grid = (unsigned)(((size_t)cbs * strips + B / 32 - 1) / (B / 32));
    if ((N & 3) == 0)
      return launch_k(stencil_kernel<B, 4>, dim3(grid), dim3(B), 0, s, a.pdl, (const float*)e.in0, (float*)e.out, N, cbs);
    return launch_k(stencil_kernel<B, 1>, dim3(grid), dim3(B), 0, s, a.pdl, (const float*)e.in0, (float*)e.out, N, cbs);
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
  static cudaError_t attrs(const void** f, size_t* sm) { return kernel_attrs(spin_kernel<B>, 0, f, sm); }
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
