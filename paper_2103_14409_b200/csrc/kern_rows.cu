// kern_rows.cu — row kernels of the suite: euclidean_kernel, matvec, rowsum.
//
// euclidean_kernel is the one kernel the paper names (Figs. 3/5).  Its source is
// not given; this build reads it as the distance of every row of A to a query vector q
// (reading R-14).  Mapping: each warp of a CTA of B threads reduces
// one row (team size 1, calibrated; larger teams remain for calibration), 128-bit streaming
// loads of A with U = 8 independent loads in flight per thread (64-register budget), q/x
// through the read-only cache (L2/L1 resident), fp32 accumulation, warp shuffles (+ a
// fixed-order smem combine for teams > 1); A's loads carry a fractional L2 evict-last policy
// (re-read by every launch of a bracket: all of A stays L2-resident when it fits, a stable
// fraction of it otherwise).  HBM bound: 4N^2 + 8N bytes per launch (fewer from DRAM in a
// bracket: the L2-resident part).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

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
#ifndef ROW_PERSIST_BIG
#define ROW_PERSIST_BIG 1  // persistent grid for B > 512 (calibration switch)
#endif
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
// UL = float4 loads of A in flight per thread per pass.  Large N: ROW_U (8) under a 64-register
// budget; short rows (a launch is latency bound: one or two passes) use lighter variants without
// the register budget -- 2-deep up to N = 256, 4-deep up to 2048.  Interleaved A/B
// (scripts/ab_small_rows.sh, plain graph brackets, mean over the 32 blocks): N = 64 2.10 ->
// 1.72 us, 256 2.23 -> 1.94, 512 2.37 -> 2.02, 1024 2.68 -> 2.63, 2048 4.08 -> 3.97
// (scripts/launch_floor_probe*.cu: an empty graph launch is 0.44 us).
constexpr int kSmallRowN = 2048;
template <int UL, int B>
constexpr int row_bounds_min_blocks() { return UL >= 8 ? row_min_blocks<B>() : 1; }

template <int OP, int B, int UL>
__global__ void __launch_bounds__(B, row_bounds_min_blocks<UL, B>()) row_kernel(const float* __restrict__ A,
                                                const float* __restrict__ v,
                                                float* __restrict__ out, int N, int TW, float l2keep) {
  constexpr int W = B / 32;
  __shared__ float red[W];
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / TW, tw = warp % TW;          // team index, warp within team
  const int T = TW * 32, t = tw * 32 + lane;            // team size, thread within team
  const int teams = W / TW;                            // warps beyond teams*TW idle
  // grid-stride over row blocks with a CTA-uniform trip count (the team combine's
  // __syncthreads is reached by every warp); the launcher makes the grid persistent for
  // B > 512 (one CTA per SM: no CTA retire/launch gaps inside a launch), one pass otherwise.
  // scripts/row_persist_probe.sh (PDL brackets, blocks 544..1024): N = 8192 34.75 -> 33.42 us,
  // N = 4096 7.00 -> 6.77 us.
  for (int row0 = blockIdx.x * teams; row0 < N; row0 += gridDim.x * teams) {
    const int row = row0 + team;
    const bool live = team < teams && row < N;
    const float* a = A + (size_t)(live ? row : 0) * N;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
      if ((N & 3) == 0) {
        constexpr int U = UL;
        const uint64_t pol = l2keep > 0.f ? l2_keep_fraction_policy(l2keep) : 0;
        const float4* a4 = reinterpret_cast<const float4*>(a);
        const float4* v4 = reinterpret_cast<const float4*>(v);
        const int n4 = N >> 2;
        for (int base = t; base < n4; base += U * T) {
          float4 x[U], y[U];
#pragma unroll
          for (int u = 0; u < U; u++) {
            const int j = base + u * T;
            x[u] = j < n4 ? (l2keep > 0.f ? ld_keep(a4 + j, pol) : ld_stream(a4 + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
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
      __syncthreads();  // red[] is rewritten by the next row block
    }
    pdl_wait();
    if (live && tw == 0 && lane == 0) out[row] = (OP == kEuclid) ? sqrtf(r) : r;
  }
}

// Warps per team (one row per team).  B200 calibration with the 64-register budget and PDL
// brackets (scripts/row_variants.sh, scripts/tw_probe.sh; euclid, mean per-launch time over
// the 32 blocks): one warp per row is best at every N -- N = 8192: 44.0 us (two-warp teams
// 45.2); N = 4096: 10.2 (10.7); N = 2048: 1.94 us (2: 2.75, 4: 4.49, the previous wave-tail
// heuristic 2.87); N = 1024: 0.83 (1.30, 2.29, heuristic 1.32); N = 512: 0.73 (0.76, 1.20).
// Larger teams only add the team combine and idle leftover warps.
inline int team_warps(int /*N*/, int /*B*/) { return 1; }

inline int small_rows() {  // LSCAT_ROW_SMALL=0: the 8-deep variant at every N; =2 also the
  static const int v = [] {  // 4-deep one up to kSmallRowN (A/B runs)
    const char* e = getenv("LSCAT_ROW_SMALL");
    return e ? atoi(e) : 2;
  }();
  return v;
}

inline int small4_max() {  // LSCAT_ROW_SMALL4_MAX: largest N of the 4-deep variant (calibration)
  static const int v = [] {
    const char* e = getenv("LSCAT_ROW_SMALL4_MAX");
    return e ? atoi(e) : 2048;
  }();
  return v;
}

inline bool legacy_grid() {
  static const bool v = [] {
    const char* e = getenv("LSCAT_ROW_GRID");
    return e && strcmp(e, "legacy") == 0;
  }();
  return v;
}

template <int OP>
struct RowLauncher {
  template <int B>
  struct L {
    static constexpr bool kSupported = true;
    static cudaError_t attrs(const void** f, size_t* sm) { return kernel_attrs(row_kernel<OP, B, ROW_U>, 0, f, sm); }
    // resident CTAs per SM of the UL variant (a property of the sm_100a binary; thread-safe
    // one-time query)
    template <int UL>
    static int per_sm_v() {
      static const int v = [] {
        int r = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, row_kernel<OP, B, UL>, B, 0);
        cudaGetLastError();
        return r > 0 ? r : 1;
      }();
      return v;
    }
    static int per_sm() { return per_sm_v<ROW_U>(); }
    static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
      const SuiteEntry& e = *a.e;
      const int N = (int)e.n;
      // calibration overrides (profiling only): LSCAT_ROW_TEAM_WARPS, LSCAT_ROW_L2FRAC
      static const int tw_env = [] {
        const char* v = getenv("LSCAT_ROW_TEAM_WARPS");
        return v ? atoi(v) : 0;
      }();
      static const double keep_env = [] {  // share of L2 the kept part of A may fill
        const char* v = getenv("LSCAT_ROW_L2FRAC");
        return v ? atof(v) : -1.0;
      }();
      const int tw = (tw_env > 0 && tw_env <= B / 32) ? tw_env : team_warps(N, B);
      const int teams = B / 32 / tw;
      // L2 residency: every launch of a bracket re-reads A.  Its loads carry a fractional L2
      // policy: an address-hashed fraction f of A's lines is kept evict-last, the rest streams
      // evict-first, with f = min(1, share x L2 / |A|), share = 0.45 (LSCAT_ROW_L2FRAC
      // overrides; 0 = plain streaming loads).  So A stays wholly L2-resident at N <= 4096
      // and a stable 21 % of it (57 MB) at N = 8192 instead of the whole L2 thrashing.
      // Measured (scripts/l2frac_probe.sh, PDL brackets, mean over the 32 blocks): N = 8192
      // share 0: 38.1 us, 0.3: 33.0, 0.45: 32.2, 0.6: 33.1, 0.75: 36.2; N = 4096: 6.2-6.3 us.
      const double share = keep_env >= 0 ? keep_env : 0.45;
      const double a_bytes = (double)N * N * 4.0;
      // LSCAT_L2_ROTATE (a.cold): plain streaming loads, nothing is kept for the next launch
      const float keep = (share <= 0 || a.cold) ? 0.f : (float)std::min(1.0, share * (double)a.l2_bytes / a_bytes);
      const int sms = a.sms > 0 ? a.sms : 148;
      // Grid: one row block per CTA while they all fit in one wave; otherwise r = ceil(row
      // blocks / resident CTAs) row blocks per CTA over the fewest CTAs that need no more than
      // r -- every CTA (and warp) streams the same number of rows and none idles through a
      // partial last round (LSCAT_ROW_GRID=legacy: the round-1 grid, for A/B runs).
      const int sv = small_rows();
      const int ul = (N <= 256 && sv) ? 2 : (N <= small4_max() && sv >= 2) ? 4 : ROW_U;
      const long need = (N + teams - 1) / teams;
      const long slots = (long)sms * (ul == 2 ? per_sm_v<2>() : ul == 4 ? per_sm_v<4>() : per_sm());
      int grid;
      if (legacy_grid()) {
        grid = (int)((ROW_PERSIST_BIG && B > 512 && need > sms) ? sms : need);
      } else if (need <= slots) {
        grid = (int)need;
      } else {
        const long r = (need + slots - 1) / slots;
        grid = (int)((need + r - 1) / r);
      }
      if (ul == 2)  // latency-bound short rows: the lighter variants
        return launch_k(row_kernel<OP, B, 2>, dim3(grid), dim3(B), 0, s, a.pdl,
                        (const float*)e.in0, (const float*)e.in1, (float*)e.out, N, tw, keep);
      if (ul == 4)
        return launch_k(row_kernel<OP, B, 4>, dim3(grid), dim3(B), 0, s, a.pdl,
                        (const float*)e.in0, (const float*)e.in1, (float*)e.out, N, tw, keep);
      return launch_k(row_kernel<OP, B, ROW_U>, dim3(grid), dim3(B), 0, s, a.pdl,
                      (const float*)e.in0, (const float*)e.in1, (float*)e.out, N, tw, keep);
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
