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

// Segments of 256 float4 per row (one pass of 8 float4 per lane of a warp), <= 32.
inline int row_segments(int N) { return (N & 3) == 0 ? std::max(1, ((N >> 2) + 255) / 256) : 1; }
inline size_t row_part_bytes(int N) { return ((size_t)N * row_segments(N) * sizeof(float) + 7) & ~(size_t)7; }
inline unsigned long long* row_tickets(const SuiteEntry& e) {
  return reinterpret_cast<unsigned long long*>((char*)e.scratch + row_part_bytes((int)e.n));
}

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

// Work split.  With at least one warp per row (N <= Wt warps in the grid) warp
// w reduces the whole rows [w N / Wt, (w+1) N / Wt).  With fewer warps than rows, rows are cut
// into S = ceil(N/4 / 256) segments of 256 float4 (one pass of 8 float4 per lane), the work
// units are the U = N S (row, segment) pairs, and warp w takes the contiguous units
// [w U / Wt, (w+1) U / Wt): every warp gets the same work to within one segment, whatever the
// block size (one row per warp left most warps idle through a second row's time: N = 8192 is
// 1.73 rows per warp at 4736 resident warps; measured 33.6-40.7 us across the blocks).
// A row a warp covers whole is reduced in registers and stored.  A row split between warps
// leaves one partial sum per piece in part[row][first segment] and adds (segments |
// 1 << (32 + first segment)) to the row's 64-bit ticket with an acq_rel atomic; the warp whose
// add completes the S segments sums the pieces in segment order, applies the finish (sqrt for
// euclid), stores the row and resets the ticket.  The atomic's result is only inspected after
// the warp's next piece has been loaded, so its round trip overlaps the streaming.
__device__ __forceinline__ unsigned long long atom_add_acq_rel(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

template <int OP>
__device__ __forceinline__ float row_finish(float s) { return OP == kEuclid ? sqrtf(s) : s; }

template <int OP, int B>
__global__ void __launch_bounds__(B, row_min_blocks<B>()) row_kernel(const float* __restrict__ A,
                                                const float* __restrict__ v,
                                                float* __restrict__ out, int N, int S, int split,
                                                float* __restrict__ part,
                                                unsigned long long* __restrict__ tick,
                                                float l2keep) {
  constexpr int W = B / 32;
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const uint64_t Wt = (uint64_t)gridDim.x * W;
  const uint64_t w = (uint64_t)blockIdx.x * W + (threadIdx.x >> 5);
  // unit = a segment when split, else a whole row
  const uint64_t U = split ? (uint64_t)N * S : (uint64_t)N;
  const int upr = split ? S : 1;  // units per row
  uint64_t u = w * U / Wt;
  const uint64_t u1 = (w + 1) * U / Wt;
  const bool vec = (N & 3) == 0;
  const int n4 = N >> 2;
  const uint64_t pol = (vec && l2keep > 0.f) ? l2_keep_fraction_policy(l2keep) : 0;
  const float4* A4 = reinterpret_cast<const float4*>(A);
  const float4* v4 = reinterpret_cast<const float4*>(v);
  int pend_r = -1;                 // split row whose ticket result is not yet inspected
  unsigned long long pend_now = 0;
  while (u < u1) {
    const int r = (int)(u / upr), p0 = (int)(u % upr);
    const int p1 = (int)min((uint64_t)upr, (uint64_t)p0 + (u1 - u));  // this piece: units [p0, p1)
    const int s0 = split ? p0 : 0, s1 = split ? p1 : S;                // segments [s0, s1)
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (vec) {
      constexpr int UL = ROW_U;  // 8 float4 per lane in flight = one 256-float4 segment
      const float4* a = A4 + (size_t)r * n4;
      for (int sg = s0; sg < s1; sg++) {
        const int base = sg * 256 + lane;
        float4 x[UL], y[UL];
#pragma unroll
        for (int k = 0; k < UL; k++) {
          const int j = base + 32 * k;
          x[k] = j < n4 ? (l2keep > 0.f ? ld_keep(a + j, pol) : ld_stream(a + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if constexpr (OP != kRowsum) {
#pragma unroll
          for (int k = 0; k < UL; k++) {
            const int j = base + 32 * k;
            y[k] = j < n4 ? __ldg(v4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int k = 0; k < UL; k++) acc4<OP>(acc, x[k], OP != kRowsum ? y[k] : x[k]);
      }
    } else {  // scalar rows (S == 1, never split)
      const float* a = A + (size_t)r * N;
      for (int j = lane; j < N; j += 32) acc.x = acc1<OP>(acc.x, ld_stream(a + j), OP != kRowsum ? __ldg(v + j) : 0.f);
    }
    float sum = (acc.x + acc.y) + (acc.z + acc.w);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    pdl_wait();  // the predecessor launch is complete before this launch's first store
    if (lane == 0) {
      if (pend_r >= 0 && (uint32_t)pend_now == (uint32_t)S) {  // the previous piece completed its row
        float tot = 0.f;
        for (uint32_t m = (uint32_t)(pend_now >> 32); m; m &= m - 1)
          tot += __ldcg(&part[(size_t)pend_r * S + (__ffs(m) - 1)]);
        out[pend_r] = row_finish<OP>(tot);
        tick[pend_r] = 0;
      }
      pend_r = -1;
      if (s0 == 0 && s1 == S) {
        out[r] = row_finish<OP>(sum);
      } else {
        part[(size_t)r * S + s0] = sum;
        const unsigned long long add = (unsigned long long)(s1 - s0) | (1ull << (32 + s0));
        pend_now = atom_add_acq_rel(&tick[r], add) + add;
        pend_r = r;
      }
    }
    u += p1 - p0;
  }
  if (lane == 0 && pend_r >= 0 && (uint32_t)pend_now == (uint32_t)S) {
    float tot = 0.f;
    for (uint32_t m = (uint32_t)(pend_now >> 32); m; m &= m - 1)
      tot += __ldcg(&part[(size_t)pend_r * S + (__ffs(m) - 1)]);
    out[pend_r] = row_finish<OP>(tot);
    tick[pend_r] = 0;
  }
}

template <int OP>
struct RowLauncher {
  template <int B>
  struct L {
    static constexpr bool kSupported = true;
    static cudaError_t attrs(const void** f, size_t* sm) { return kernel_attrs(row_kernel<OP, B>, 0, f, sm); }
    // resident CTAs per SM (a property of the sm_100a binary; thread-safe one-time query)
    static int per_sm() {
      static const int v = [] {
        int r = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, row_kernel<OP, B>, B, 0);
        cudaGetLastError();
        return r > 0 ? r : 1;
      }();
      return v;
    }
    static cudaError_t launch(const LaunchArgs& a, cudaStream_t s) {
      const SuiteEntry& e = *a.e;
      const int N = (int)e.n;
      // calibration override (profiling only): LSCAT_ROW_L2FRAC
      static const double keep_env = [] {  // share of L2 the kept part of A may fill
        const char* v = getenv("LSCAT_ROW_L2FRAC");
        return v ? atof(v) : -1.0;
      }();
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
      const int S = row_segments(N);
      // one row per warp at most (small N: the launch is latency bound), else all resident
      // warps of the device, with the units spread evenly over them
      const long need = (N + B / 32 - 1) / (B / 32);
      const int grid = (int)std::min<long>(need, (long)per_sm() * sms);
      const int split = (long)grid * (B / 32) < N && S > 1;  // fewer warps than rows
      return launch_k(row_kernel<OP, B>, dim3(grid), dim3(B), 0, s, a.pdl,
                      (const float*)e.in0, (const float*)e.in1, (float*)e.out, N, S, split,
                      (float*)e.scratch, row_tickets(e), keep);
    }
  };
};

template <int B> using EuclidL = RowLauncher<kEuclid>::L<B>;
template <int B> using MatvecL = RowLauncher<kMatvec>::L<B>;
template <int B> using RowsumL = RowLauncher<kRowsum>::L<B>;

}  // namespace

// Split-row partials [N][S] and per-row tickets [N] (zero; the completing warp re-zeroes its
// row's ticket, so consecutive launches need no reset).
cudaError_t row_prepare(SuiteEntry& e) {
  if (e.n > 32768) return cudaErrorInvalidValue;  // S <= 32 segments (ticket bit mask)
  e.scratch_bytes = row_part_bytes((int)e.n) + (size_t)e.n * sizeof(unsigned long long);
  cudaError_t err = cudaMalloc(&e.scratch, e.scratch_bytes);
  if (err != cudaSuccess) return err;
  return cudaMemset(e.scratch, 0, e.scratch_bytes);
}

const KernelTable& table_euclid() { static KernelTable t = make_table<EuclidL>(); return t; }
const KernelTable& table_matvec() { static KernelTable t = make_table<MatvecL>(); return t; }
const KernelTable& table_rowsum() { static KernelTable t = make_table<RowsumL>(); return t; }

}  // namespace lscat
