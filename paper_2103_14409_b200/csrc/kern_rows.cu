// kern_rows.cu — row kernels of the suite: euclidean_kernel, matvec, rowsum.
//
// euclidean_kernel is the one kernel the paper names (Figs. 3/5).  Its source is
// not given; this build reads it as the distance of every row of A to a query vector q
// (reading R-14).  Mapping: one CTA of B threads per row, 128-bit
// streaming loads of A with U independent loads in flight per thread, q/x through the
// read-only cache (L2/L1 resident), fp32 accumulation, warp-shuffle + shared-memory tree.
// HBM bound: 4N^2 + 8N bytes per launch.
#include "kern_common.cuh"

namespace lscat {
namespace {

enum RowOp { kEuclid = 0, kMatvec = 1, kRowsum = 2 };

template <int OP>
__device__ __forceinline__ void acc4(float4& s, float4 a, float4 v) {
  if constexpr (OP == kEuclid) {
    float d0 = a.x - v.x, d1 = a.y - v.y, d2 = a.z - v.z, d3 = a.w - v.w;
    s.x = fmaf(d0, d0, s.x); s.y = fmaf(d1, d1, s.y); s.z = fmaf(d2, d2, s.z); s.w = fmaf(d3, d3, s.w);
  } else if constexpr (OP == kMatvec) {
    s.x = fmaf(a.x, v.x, s.x); s.y = fmaf(a.y, v.y, s.y); s.z = fmaf(a.z, v.z, s.z); s.w = fmaf(a.w, v.w, s.w);
  } else {
    s.x += a.x; s.y += a.y; s.z += a.z; s.w += a.w;
  }
}

template <int OP>
__device__ __forceinline__ float acc1(float s, float a, float v) {
  if constexpr (OP == kEuclid) { float d = a - v; return fmaf(d, d, s); }
  else if constexpr (OP == kMatvec) return fmaf(a, v, s);
  else return s + a;
}

template <int OP, int B>
__global__ void __launch_bounds__(B) row_kernel(const float* __restrict__ A,
                                                const float* __restrict__ v,
                                                float* __restrict__ out, int N) {
  __shared__ float red[B / 32 > 0 ? B / 32 : 1];
  const float* a = A + (size_t)blockIdx.x * N;
  const int t = threadIdx.x;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if ((N & 3) == 0) {
    constexpr int U = 4;
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* v4 = reinterpret_cast<const float4*>(v);
    const int n4 = N >> 2;
    for (int base = t; base < n4; base += U * B) {
      float4 x[U], y[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int j = base + u * B;
        x[u] = j < n4 ? ld_stream(a4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if constexpr (OP != kRowsum) {
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int j = base + u * B;
          y[u] = j < n4 ? __ldg(v4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) acc4<OP>(s, x[u], OP != kRowsum ? y[u] : x[u]);
    }
  } else {
    for (int j = t; j < N; j += B) s.x = acc1<OP>(s.x, ld_stream(a + j), OP != kRowsum ? __ldg(v + j) : 0.f);
  }
  float r = block_sum<B>((s.x + s.y) + (s.z + s.w), red);
  if (t == 0) out[blockIdx.x] = (OP == kEuclid) ? sqrtf(r) : r;
}

template <int OP>
struct RowLauncher {
  template <int B>
  struct L {
    static constexpr bool kSupported = true;
    static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
      const SuiteEntry& e = *a.e;
      row_kernel<OP, B><<<e.n, B, 0, s>>>((const float*)e.in0, (const float*)e.in1,
                                          (float*)e.out, (int)e.n);
      return cudaGetLastError();
    }
  };
};

template <int B> using EuclidL = RowLauncher<kEuclid>::L<B>;
template <int B> using MatvecL = RowLauncher<kMatvec>::L<B>;
template <int B> using RowsumL = RowLauncher<kRowsum>::L<B>;

}  // namespace

const KernelTable& table_euclid() { static KernelTable t = make_table<EuclidL>(); return t; }
const KernelTable& table_matvec() { static KernelTable t = make_table<MatvecL>(); return t; }
const KernelTable& table_rowsum() { static KernelTable t = make_table<RowsumL>(); return t; }

}  // namespace lscat
