// kern_rows.cu — row kernels of the suite: euclidean_kernel, matvec, rowsum.
//
// euclidean_kernel is the one kernel the paper names (Figs. 3/5).  Its source is
// not given; this build reads it as the distance of every row of A to a query vector q
// (reading R-14).  Mapping: a CTA of B threads is split into teams of
// warps, one team per row (one team per CTA for small blocks or long rows), 128-bit streaming
// loads of A with U independent loads in flight per thread, q/x through the read-only cache
// (L2/L1 resident), fp32 accumulation, warp shuffles + a fixed-order smem combine.
// HBM bound: 4N^2 + 8N bytes per launch.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "kern_common.cuh"

namespace lscat {
namespace {

enum RowOp { kEuclid = 0, kMatvec = 1, kRowsum = 2 };

#ifndef ROW_U
#define ROW_U 8  // float4 loads of A in flight per thread (and as many of q/x)
#endif
// Register budget: ptxas otherwise sizes registers for full occupancy (32 regs for B >= 64),
// which serialises the U loads (one 128-bit load in flight per thread).  Declaring at least
// ROW_MINB_THREADS / B resident CTAs caps registers at 65536 / ROW_MINB_THREADS instead
// (scripts/row_variants.sh: 1024 -> 64 registers is best on B200).
#ifndef ROW_MINB_THREADS
#define ROW_MINB_THREADS 1024
#endif
template <int B>
constexpr int row_min_blocks() { return ROW_MINB_THREADS / B > 0 ? ROW_MINB_THREADS / B : 1; }

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

// A CTA of B threads is split into floor(W/TW) teams of TW warps; each team reduces one row
// (TW from team_warps, calibrated on B200).
template <int OP, int B>
__global__ void __launch_bounds__(B, row_min_blocks<B>()) row_kernel(const float* __restrict__ A,
                                                const float* __restrict__ v,
                                                float* __restrict__ out, int N, int TW) {
  constexpr int W = B / 32;
  __shared__ float red[W];
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / TW, tw = warp % TW;          // team index, warp within team
  const int T = TW * 32, t = tw * 32 + lane;            // team size, thread within team
  const int teams = W / TW;                            // warps beyond teams*TW idle
  const int row = blockIdx.x * teams + team;
  const bool live = team < teams && row < N;
  const float* a = A + (size_t)(live ? row : 0) * N;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (live) {
    if ((N & 3) == 0) {
      constexpr int U = ROW_U;
      const float4* a4 = reinterpret_cast<const float4*>(a);
      const float4* v4 = reinterpret_cast<const float4*>(v);
      const int n4 = N >> 2;
      for (int base = t; base < n4; base += U * T) {
        float4 x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int j = base + u * T;
          x[u] = j < n4 ? ld_stream(a4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if constexpr (OP != kRowsum) {
#pragma unroll
          for (int u = 0; u < U; u++) {
            const int j = base + u * T;
            y[u] = j < n4 ? __ldg(v4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < U; u++) acc4<OP>(s, x[u], OP != kRowsum ? y[u] : x[u]);
      }
    } else {
      for (int j = t; j < N; j += T) s.x = acc1<OP>(s.x, ld_stream(a + j), OP != kRowsum ? __ldg(v + j) : 0.f);
    }
  }
  float r = (s.x + s.y) + (s.z + s.w);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  if (TW > 1) {  // combine the team's warps in a fixed order
    if (lane == 0) red[warp] = r;
    __syncthreads();
    if (tw == 0 && lane == 0) {
      r = 0.f;
      if (team < teams)
        for (int k = 0; k < TW; k++) r += red[team * TW + k];
    }
  }
  pdl_wait();
  if (live && tw == 0 && lane == 0) out[row] = (OP == kEuclid) ? sqrtf(r) : r;
}

// Warps per team d (1..W, W = B/32; floor(W/d) teams per CTA, leftover warps idle).
// B200 calibration (profiles/r01_summary.md, scripts/row_variants.sh; euclid, U = 8, 64
// registers): at N >= 4096 one warp per row is best at every block (N = 8192: mean over the
// 32 blocks 44.0 us vs 45.2 for two-warp teams; N = 4096: 10.2 vs 10.7).  Smaller matrices
// have fewer rows than resident warps, so teams split rows to fill the machine; the score
// there = active fraction x preference(d) x wave-tail penalty.
inline int team_warps(int N, int B, int sm_count, int resident) {
  const int W = B / 32;
  if (N >= 4096) return 1;
  const double slots = (double)sm_count * resident;
  int best = 1;
  double best_score = -1.0;
  for (int d = 1; d <= W; d++) {
    const int teams = W / d;
    const double pref = d == 2 ? 1.0 : (d == 3 || d == 4) ? 0.99 : d == 1 ? 0.96 : (d <= 8 ? 0.97 : 0.93);
    const double active = (double)(teams * d) / W;
    const double waves = std::ceil((double)N / teams) / slots;
    const double tail = (waves > 1.0 && waves < 1.3) ? 0.5 : (waves > 2.0 && waves < 2.3) ? 0.8 : 1.0;
    const double score = active * pref * tail;
    if (score > best_score + 1e-9) { best_score = score; best = d; }
  }
  return best;
}

template <int OP>
struct RowLauncher {
  template <int B>
  struct L {
    static constexpr bool kSupported = true;
    static int occupancy() { return occupancy_warps(row_kernel<OP, B>, B); }
    static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
      const SuiteEntry& e = *a.e;
      // CTAs resident per SM from threads (2048), CTAs (32) and registers (64K, allocated per
      // warp in units of 256); shared memory (< 1 KB) never binds
      static int sm_count = 0, resident = 0;
      if (!resident) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
        if (sm_count < 1) sm_count = 148;
        cudaFuncAttributes fa{};
        int regs = 32;
        if (cudaFuncGetAttributes(&fa, row_kernel<OP, B>) == cudaSuccess && fa.numRegs > 0) regs = fa.numRegs;
        cudaGetLastError();
        const int per_warp = ((regs * 32 + 255) / 256) * 256;
        resident = std::max(1, std::min({32, 2048 / B, 65536 / (per_warp * (B / 32))}));
      }
      // tuning overrides (profiling only): LSCAT_ROW_TEAM_WARPS, LSCAT_ROW_WARPS_PER_SM
      static const int tw_env = [] {
        const char* v = getenv("LSCAT_ROW_TEAM_WARPS");
        return v ? atoi(v) : 0;
      }();
      static const int cap_env = [] {
        const char* v = getenv("LSCAT_ROW_WARPS_PER_SM");
        return v ? atoi(v) : -1;
      }();
      // Optional cap on resident warps per SM by reserving dynamic shared memory (calibration
      // only, off by default: the reservation also shrinks L1, which holds q/x, and measured
      // slower on B200 for every cap tried, profiles/r01_summary.md).
      static int smem_cap = -1;
      if (smem_cap < 0) {
        const int cap = cap_env >= 0 ? cap_env : 0;
        const int W = B / 32;
        smem_cap = 0;
        if (cap > 0 && resident * W > cap) {
          const int ctas = std::max(1, cap / W);
          smem_cap = (227 * 1024) / ctas - 1024;  // leaves room for the static red[] array
          smem_cap = std::min(smem_cap, 227 * 1024 - 2048);
          if (cudaFuncSetAttribute(row_kernel<OP, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap) !=
              cudaSuccess) {
            cudaGetLastError();
            smem_cap = 0;
          } else {
            resident = ctas;
          }
        }
      }
      const int N = (int)e.n;
      const int tw = (tw_env > 0 && tw_env <= B / 32) ? tw_env : team_warps(N, B, sm_count, resident);
      const int teams = B / 32 / tw;
      return launch_k(row_kernel<OP, B>, dim3((N + teams - 1) / teams), dim3(B), (size_t)smem_cap, s, a.pdl,
                      (const float*)e.in0, (const float*)e.in1, (float*)e.out, N, tw);
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
