// reduce.cu — a6 (per-group reduce), a7 (global accumulate), a9 (NCCL merge) and
// a8/a10 (percentile selection, finalize) of the runtime-table analysis.
//
// The paper's statistics are group-wise: per (kernel, matrix size)
// slice, the best block, the largest (1024) block's performance b/t and the optimal block's
// gain t/b - 1; then shares, means and histograms over slices.  DESIGN.md §4 lists the exact
// definitions (readings R-4..R-13) this kernel implements; the integer outputs (argmin ids,
// counts, histograms, fixed-point sums) are exact and order independent, so they are
// bit-identical to the CPU oracle and across shard counts.
//
// Kernel layout: persistent grid, a warp takes 32 consecutive groups at a
// time and lane j ends up owning group j.  Three ways to get there:
//   * uniform 32-row tables (configs[4]): cp.async 16-byte copies into an XOR-swizzled warp
//     stage, lane j folds group j in one pass when its block ids are 0..31 in order (first
//     minimum = smallest id among equal minima; positive finite fp32 bit patterns order like
//     their values), else a second pass over the ids; the next batch streams in while this
//     one is finalised;
//   * ragged tables with groups of <= 32 rows: coalesced loads into a padded stage, lane j
//     folds group j's rows;
//   * longer groups: the warp folds each group with redux.sync.min / ballots.
// The 32 lanes then finalise their groups in parallel (f64 ratios, exact bins, flags) into
// shared-memory histograms and CTA counters, flushed once per CTA with 64-bit atomics.
// HBM: 6 B/row read (+16 B/group of perf/gain written).
#include <algorithm>
#include <map>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.h"

namespace lscat {
namespace {

enum { MODE_FUSED = 0, MODE_GROUP_PARTIALS = 1, MODE_FINALIZE_MERGED = 2 };
constexpr int kNC = LSCAT_P_NCOUNTERS;

struct RP {
  const float* rt;
  const uint16_t* bid;
  const int64_t* off;
  const uint32_t* gmat;
  uint64_t n_groups, first_group;
  uint32_t rpg;
  uint64_t n_rows;
  uint32_t L, ell, M, policy, nb, cap;
  uint32_t ggn, ggd, pln, pld, bln, bld;
  // per-group outputs (may be null)
  uint16_t* o_best;
  float* o_bestrt;
  double* o_perf;
  double* o_gain;
  uint32_t* o_flags;
  // accumulation
  uint64_t* partials;
  uint64_t* minmax;  // [4] perf min/max key, gain min/max key over accumulated groups
  uint64_t acc_lo, acc_hi;
  // point-sharded merge arrays
  uint64_t* g_key;
  uint64_t* g_lcode;
  uint32_t* g_cnt;  // [3*G]: n_ok, n_nan, n_rows
  int mode;
  // per-kernel roll-up (R-26): per-group record fx_perf | rd << 53 | not_best << 54
  uint64_t* krec;
  uint32_t smem_words;  // perf + gain + best-block histogram words in smem
  uint32_t vec;         // runtime / block-id arrays are 16-byte aligned (vector path allowed)
};

struct GroupAcc {
  uint32_t min_bits, min_bid;  // 0xFFFFFFFF if no ok row
  uint32_t n_ok, n_nan, n_rows;
  uint32_t lcode;  // 0 absent, 1 present but no result, 2 present with a result
  uint32_t l_bits;
};

// Per-warp accumulators.  Counters are warp-uniform (built from ballots / redux, identical in
// every lane, flushed by lane 0); fixed-point sums and percentile key bounds are per lane.
struct ThreadAcc {
  uint64_t fx[4];                  // perf hi, perf lo, gain hi, gain lo
  uint64_t pmin, pmax, gmin, gmax;
  // Per-lane counters since the last flush_counters (every kPkGroups groups per lane): 15
  // packed 4-bit fields (the 12 flag counters LSCAT_P_GROUPS.., the perf == 1 and gain == 0
  // histogram bins, LSCAT_P_BAD_IDS) and the row counts (groups of < 2^28 rows).
  uint64_t pk;
  uint32_t rows, ok, nan;
  uint32_t n;                      // groups finalised since the last flush (warp-uniform)
};
constexpr uint32_t kPkGroups = 15;  // 4-bit fields: at most 15 increments between flushes

__device__ __forceinline__ bool ok_bits(uint32_t b) { return b - 1u < 0x7F7FFFFFu; }  // 0 < b < 0x7F800000
__device__ __forceinline__ bool nan_bits(uint32_t b) { return (b & 0x7FFFFFFFu) > 0x7F800000u; }

__device__ __forceinline__ void acc_init(GroupAcc& a) {
  a.min_bits = a.min_bid = 0xFFFFFFFFu;
  a.n_ok = a.n_nan = a.n_rows = 0;
  a.lcode = 0;
  a.l_bits = 0;
}

// One row folded into a lane's own accumulator (staged path: one group per lane).
__device__ __forceinline__ void fold_row(GroupAcc& a, uint32_t bits, uint32_t b, uint32_t ell) {
  const bool ok = ok_bits(bits);
  a.n_rows++;
  a.n_ok += ok;
  a.n_nan += nan_bits(bits);
  if (ok && (bits < a.min_bits || (bits == a.min_bits && b < a.min_bid))) {
    a.min_bits = bits;
    a.min_bid = b;
  }
  if (b == ell) {
    a.lcode = ok ? 2u : 1u;
    a.l_bits = bits;
  }
}

// Fold one chunk of <= 32 rows (lane-distributed) into a warp-uniform accumulator (fallback
// path for groups of more than 32 rows).
__device__ __forceinline__ void fold_chunk(GroupAcc& a, bool valid, uint32_t bits, uint32_t b,
                                           uint32_t ell) {
  const unsigned FULL = 0xffffffffu;
  const bool ok = valid && ok_bits(bits);
  const uint32_t m = __reduce_min_sync(FULL, ok ? bits : 0xFFFFFFFFu);
  const uint32_t mb = __reduce_min_sync(FULL, (ok && bits == m) ? b : 0xFFFFFFFFu);
  if (m < a.min_bits || (m == a.min_bits && mb < a.min_bid)) { a.min_bits = m; a.min_bid = mb; }
  a.n_ok += __popc(__ballot_sync(FULL, ok));
  a.n_nan += __popc(__ballot_sync(FULL, valid && nan_bits(bits)));
  a.n_rows += __popc(__ballot_sync(FULL, valid));
  const unsigned lb = __ballot_sync(FULL, valid && b == ell);
  if (lb) {
    const uint32_t lbits = __shfl_sync(FULL, bits, __ffs(lb) - 1);
    a.lcode = ok_bits(lbits) ? 2u : 1u;
    a.l_bits = lbits;
  }
}

__device__ __forceinline__ uint64_t f64_key(double v) { return (uint64_t)__double_as_longlong(v); }

__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp-collective: add the lanes' packed counters and row counts to the CTA's shared counters.
__device__ __forceinline__ void flush_counters(const RP& p, ThreadAcc& t, uint64_t* sh_c, uint32_t* sh_perf,
                                            uint32_t* sh_gain) {
  const unsigned FULL = 0xffffffffu;
  const bool l0 = (threadIdx.x & 31) == 0;
#pragma unroll
  for (int i = 0; i < 12; i++) {
    const uint32_t v = __reduce_add_sync(FULL, (uint32_t)(t.pk >> (4 * i)) & 15u);
    if (l0 && v) atomicAdd((unsigned long long*)&sh_c[LSCAT_P_GROUPS + i], (unsigned long long)v);
  }
  const uint32_t hp = __reduce_add_sync(FULL, (uint32_t)(t.pk >> 48) & 15u);
  const uint32_t hg = __reduce_add_sync(FULL, (uint32_t)(t.pk >> 52) & 15u);
  const uint32_t bad = __reduce_add_sync(FULL, (uint32_t)(t.pk >> 56) & 15u);
  if (l0 && bad) atomicAdd((unsigned long long*)&sh_c[LSCAT_P_BAD_IDS], (unsigned long long)bad);
  if (l0 && hp) atomicAdd(&sh_perf[p.nb], hp);
  if (l0 && hg) atomicAdd(&sh_gain[0], hg);
  const uint64_t r = warp_sum64(t.rows), o = warp_sum64(t.ok), n = warp_sum64(t.nan);
  if (l0 && r) {
    atomicAdd((unsigned long long*)&sh_c[LSCAT_P_ROWS], (unsigned long long)r);
    atomicAdd((unsigned long long*)&sh_c[LSCAT_P_OK], (unsigned long long)o);
    atomicAdd((unsigned long long*)&sh_c[LSCAT_P_NAN], (unsigned long long)n);
    atomicAdd((unsigned long long*)&sh_c[LSCAT_P_INVALID], (unsigned long long)(r - o - n));
  }
  t.pk = 0;
  t.rows = t.ok = t.nan = 0;
  t.n = 0;
}

// The paper's per-group statistics (O3 steps 3-9).  Warp-collective: all 32
// lanes call it; `active` lanes hold group g's accumulator.
__device__ void finalize_lane(const RP& p, uint64_t g, bool active, const GroupAcc& a,
                              ThreadAcc& t, uint64_t* sh_c, uint32_t* sh_perf, uint32_t* sh_gain,
                              uint32_t* sh_bb) {
  const bool acc = active && g >= p.acc_lo && g < p.acc_hi;
  const bool complete = a.n_rows == p.L && a.n_ok == a.n_rows;
  const bool defined = active && (p.policy ? complete : a.n_ok >= 1);
  uint32_t flags = 0;
  if (a.n_ok == 0) flags |= LSCAT_GF_ALL_NAN;
  if (complete) flags |= LSCAT_GF_COMPLETE;
  double perf = __longlong_as_double(0x7FF8000000000000ll), gain = perf;
  int pbin = -1, gbin = -1, bbi = -1;
  if (defined) {
    flags |= LSCAT_GF_DEFINED;
    const uint64_t ag = p.first_group + g;  // implicit matrix index: a mask when M is a power of 2
    const uint32_t mat = p.gmat ? p.gmat[g] : (uint32_t)((p.M & (p.M - 1)) == 0 ? (ag & (p.M - 1)) : ag % p.M);
    // ids outside [0, L) x [0, M) violate the table precondition: counted, never indexed
    bbi = (a.min_bid < p.L && mat < p.M) ? (int)(mat * p.L + a.min_bid) : -2;
    if (a.lcode == 2) {
      flags |= LSCAT_GF_RATIO_DEFINED;
      const double b = (double)__uint_as_float(a.min_bits), tt = (double)__uint_as_float(a.l_bits);
      perf = __ddiv_rn(b, tt);
      gain = __dsub_rn(__ddiv_rn(tt, b), 1.0);
      if (a.min_bid == p.ell) flags |= LSCAT_GF_LARGEST_IS_BEST;
      if (tt > b) flags |= LSCAT_GF_LARGEST_SLOWER;
      // exact rational predicates: products of an fp32 value and an integer < 2^29 are exact
      if (__dmul_rn((double)p.ggd, tt) > __dmul_rn((double)(p.ggd + p.ggn), b)) flags |= LSCAT_GF_GAIN_GT;
      const bool plt = __dmul_rn((double)p.pld, b) < __dmul_rn((double)p.pln, tt);
      if (plt) flags |= LSCAT_GF_PERF_LT;
      if (plt && __dmul_rn((double)p.bld, b) >= __dmul_rn((double)p.bln, tt)) flags |= LSCAT_GF_PERF_BAND;
      if (acc) {
        const double nbb = __dmul_rn((double)p.nb, b), nbt = __dmul_rn((double)p.nb, tt);
        // perf bin: largest k with k t <= nb b (estimate from perf, then exact fix-up)
        int k = (int)floor(__dmul_rn(perf, (double)p.nb));
        while (__dmul_rn((double)(k + 1), tt) <= nbb) k++;
        while (k > 0 && __dmul_rn((double)k, tt) > nbb) k--;
        pbin = k;
        // gain bin: overflow iff t >= (cap+1) b; else m - nb, m = largest with m b <= nb t
        if (tt >= __dmul_rn((double)(p.cap + 1), b)) {
          gbin = (int)(p.cap * p.nb);
        } else {
          int m = (int)floor(__dmul_rn(__dadd_rn(gain, 1.0), (double)p.nb));
          while (__dmul_rn((double)(m + 1), b) <= nbt) m++;
          while (__dmul_rn((double)m, b) > nbt) m--;
          gbin = m - (int)p.nb;
        }
        const uint64_t fxp = (uint64_t)__dmul_rn(perf, 4503599627370496.0);  // floor(perf 2^52)
        const double gc = gain < 1048576.0 ? gain : 1048576.0;
        const uint64_t fxg = (uint64_t)__dmul_rn(gc, 4294967296.0);          // floor(gain 2^32)
        t.fx[0] += fxp >> 21;
        t.fx[1] += fxp & ((1ull << 21) - 1);
        t.fx[2] += fxg >> 21;
        t.fx[3] += fxg & ((1ull << 21) - 1);
        const uint64_t kp = f64_key(perf), kg = f64_key(gain);
        t.pmin = min(t.pmin, kp); t.pmax = max(t.pmax, kp);
        t.gmin = min(t.gmin, kg); t.gmax = max(t.gmax, kg);
      }
    } else {
      flags |= LSCAT_GF_LARGEST_MISSING;
    }
  }
  if (active && p.krec) {  // roll-up record of an accumulated, ratio-defined group
    uint64_t r = 0;
    if (acc && (flags & LSCAT_GF_RATIO_DEFINED))
      r = (uint64_t)__dmul_rn(perf, 4503599627370496.0) | (1ull << 53) |
          ((uint64_t)((flags & LSCAT_GF_LARGEST_IS_BEST) == 0) << 54);
    p.krec[g] = r;
  }
  if (active) {
    if (p.o_best) p.o_best[g] = defined ? (uint16_t)a.min_bid : (uint16_t)0xFFFF;
    if (p.o_bestrt) p.o_bestrt[g] = defined ? __uint_as_float(a.min_bits) : __int_as_float(0x7FC00000);
    if (p.o_perf) p.o_perf[g] = perf;
    if (p.o_gain) p.o_gain[g] = gain;
    if (p.o_flags) p.o_flags[g] = flags;
  }
  // per-lane accumulation: packed flag counters and row counts, flushed every kPkGroups groups
  const bool bad_ids = acc && bbi == -2;
  if (!acc || bad_ids) bbi = -1;
  if (!acc) flags = 0;
  {
    uint64_t inc = acc ? 1ull : 0ull;  // field 0: LSCAT_P_GROUPS
    inc |= (uint64_t)((flags & LSCAT_GF_DEFINED) != 0) << 4;
    inc |= (uint64_t)((flags & LSCAT_GF_ALL_NAN) != 0) << 8;
    inc |= (uint64_t)((flags & LSCAT_GF_COMPLETE) != 0) << 12;
    inc |= (uint64_t)(acc && !(flags & LSCAT_GF_COMPLETE)) << 16;
    inc |= (uint64_t)((flags & LSCAT_GF_LARGEST_MISSING) != 0) << 20;
    inc |= (uint64_t)((flags & LSCAT_GF_RATIO_DEFINED) != 0) << 24;
    inc |= (uint64_t)((flags & LSCAT_GF_LARGEST_IS_BEST) != 0) << 28;
    inc |= (uint64_t)((flags & LSCAT_GF_LARGEST_SLOWER) != 0) << 32;
    inc |= (uint64_t)((flags & LSCAT_GF_GAIN_GT) != 0) << 36;
    inc |= (uint64_t)((flags & LSCAT_GF_PERF_LT) != 0) << 40;
    inc |= (uint64_t)((flags & LSCAT_GF_PERF_BAND) != 0) << 44;
    inc |= (uint64_t)(pbin == (int)p.nb) << 48;  // hot bins: perf == 1, gain == 0
    inc |= (uint64_t)(gbin == 0) << 52;
    inc |= (uint64_t)bad_ids << 56;
    t.pk += inc;
    if (acc) { t.rows += a.n_rows; t.ok += a.n_ok; t.nan += a.n_nan; }
  }
  if (pbin >= 0 && pbin != (int)p.nb) atomicAdd(&sh_perf[pbin], 1u);
  if (gbin > 0) atomicAdd(&sh_gain[gbin], 1u);
  if (bbi >= 0) atomicAdd(&sh_bb[bbi], 1u);
  if (++t.n == kPkGroups) flush_counters(p, t, sh_c, sh_perf, sh_gain);
}

__device__ void flush(const RP& p, ThreadAcc& t, uint64_t* sh_c, uint32_t* sh) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  if (__any_sync(FULL, t.n != 0)) flush_counters(p, t, sh_c, sh, sh + (p.nb + 1));
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint64_t v = t.fx[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    if (lane == 0 && v) atomicAdd((unsigned long long*)&sh_c[LSCAT_P_PERF_FX_HI + i], (unsigned long long)v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t.pmin = min(t.pmin, (uint64_t)__shfl_xor_sync(FULL, t.pmin, o));
    t.pmax = max(t.pmax, (uint64_t)__shfl_xor_sync(FULL, t.pmax, o));
    t.gmin = min(t.gmin, (uint64_t)__shfl_xor_sync(FULL, t.gmin, o));
    t.gmax = max(t.gmax, (uint64_t)__shfl_xor_sync(FULL, t.gmax, o));
  }
  if (lane == 0 && t.pmin <= t.pmax) {
    atomicMin((unsigned long long*)&p.minmax[0], (unsigned long long)t.pmin);
    atomicMax((unsigned long long*)&p.minmax[1], (unsigned long long)t.pmax);
    atomicMin((unsigned long long*)&p.minmax[2], (unsigned long long)t.gmin);
    atomicMax((unsigned long long*)&p.minmax[3], (unsigned long long)t.gmax);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kNC; i += blockDim.x)
    if (sh_c[i]) atomicAdd((unsigned long long*)&p.partials[i], (unsigned long long)sh_c[i]);
  for (uint32_t i = threadIdx.x; i < p.smem_words; i += blockDim.x)
    if (sh[i]) atomicAdd((unsigned long long*)&p.partials[kNC + i], (unsigned long long)sh[i]);
}

__device__ __forceinline__ void init_shared(const RP& p, uint64_t* sh_c, uint32_t* sh, ThreadAcc& t) {
  for (int i = threadIdx.x; i < kNC; i += blockDim.x) sh_c[i] = 0;
  for (uint32_t i = threadIdx.x; i < p.smem_words; i += blockDim.x) sh[i] = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) t.fx[i] = 0;
  t.pmin = t.gmin = ~0ull;
  t.pmax = t.gmax = 0;
  t.pk = 0;
  t.rows = t.ok = t.nan = 0;
  t.n = 0;
  __syncthreads();
}

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kStageRows = 1024;                      // rows staged per warp batch
constexpr int kStagePad = kStageRows + kStageRows / 32;  // + 1 word per 32 rows: no bank conflicts
constexpr size_t kStageBytes = (size_t)kWarps * kStagePad * (4 + 2);


constexpr size_t kUniStageBytes = (size_t)kWarps * (1024 * 4 + 1024 * 2);  // one stage per warp

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}

// Copy batch `base` (32 uniform groups = 1024 rows) into a warp stage buffer with cp.async:
// 8 x 16 B of runtimes and 4 x 16 B of block ids per lane, coalesced, placed in an
// XOR-swizzled layout (chunk c of group g at c ^ (g & 7) resp. c ^ ((g >> 1) & 3)) so that
// the per-group 128-bit reads below (lane j <- group j) are bank-conflict free.
__device__ __forceinline__ void uniform_prefetch_rows(const RP& p, uint64_t row0, float4* d, uint4* di, int lane) {
  const float4* src = reinterpret_cast<const float4*>(p.rt + row0);
  const uint4* isrc = reinterpret_cast<const uint4*>(p.bid + row0);
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const int f = lane + 32 * i, g = f >> 3, c = f & 7;
    cp_async16(d + g * 8 + (c ^ (g & 7)), src + f);
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int h = lane + 32 * i, g = h >> 2, c = h & 3;
    cp_async16(di + g * 4 + (c ^ ((g >> 1) & 3)), isrc + h);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void uniform_prefetch(const RP& p, uint64_t base, float4* d, uint4* di, int lane) {
  uniform_prefetch_rows(p, base * 32, d, di, lane);
}

__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr));
  return v;
}

// Lane j folds group j of a staged batch (shared-space addresses of the runtime / id stage).
__device__ __forceinline__ uint32_t lds32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

// Lane j folds group j of a staged batch (shared-space addresses of the runtime / id stage).
// Fast path when the group's block ids are 0..31 in order (every table the sweep or the
// generator writes): one pass tracks the first minimum (= the smallest block id among equal
// minima), the largest block's row is read directly.  Otherwise a second pass over ids.
__device__ __forceinline__ void uniform_fold(const RP& p, uint32_t srt, uint32_t sid, int lane,
                                             GroupAcc& mine) {
  const uint32_t rbase = srt + lane * 128, ibase = sid + lane * 64;
  const int sw = lane & 7, swi = (lane >> 1) & 3;
  bool sorted = true;
#pragma unroll
  for (int c = 0; c < 4; c++) {  // ids 8c .. 8c+7 packed in pairs: word w = (2w+1) << 16 | 2w
    const uint4 y = lds128(ibase + 16 * (c ^ swi));
    const uint32_t w0 = 8 * c;
    sorted &= y.x == (((w0 + 1) << 16) | w0) && y.y == (((w0 + 3) << 16) | (w0 + 2)) &&
              y.z == (((w0 + 5) << 16) | (w0 + 4)) && y.w == (((w0 + 7) << 16) | (w0 + 6));
  }
  uint32_t mkey = 0xFFFFFFFFu, mpos = 0xFFFFFFFFu, okm = 0;
#pragma unroll  // fully: the bit positions 4c + q of okm / mpos become constants
  for (int c = 0; c < 8; c++) {
    const uint4 x = lds128(rbase + 16 * (c ^ sw));
    const uint32_t b4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const bool ok = ok_bits(b4[q]);
      const bool lt = ok && b4[q] < mkey;  // strict: ties keep the earlier row
      mkey = lt ? b4[q] : mkey;
      mpos = lt ? (uint32_t)(4 * c + q) : mpos;
      okm |= ok ? (1u << (4 * c + q)) : 0u;
    }
  }
  uint32_t nnan = 0;
  for (uint32_t m = ~okm; m; m &= m - 1) {  // rows without a result (rare): NaN or invalid
    const int j = __ffs(m) - 1;
    nnan += nan_bits(lds32(rbase + 16 * ((j >> 2) ^ sw) + 4 * (j & 3)));
  }
  mine.min_bits = mkey;
  mine.n_ok = __popc(okm);
  mine.n_nan = nnan;
  mine.n_rows = 32;
  if (sorted) {
    mine.min_bid = mkey != 0xFFFFFFFFu ? mpos : 0xFFFFFFFFu;
    if (p.ell < 32) {
      const int j = (int)p.ell;
      const uint32_t lb = lds32(rbase + 16 * ((j >> 2) ^ sw) + 4 * (j & 3));
      mine.lcode = ok_bits(lb) ? 2u : 1u;
      mine.l_bits = lb;
    }
    return;
  }
  uint32_t mid = 0xFFFFFFFFu;
#pragma unroll 1
  for (int c = 0; c < 4; c++) {
    const uint4 y = lds128(ibase + 16 * (c ^ swi));
    const uint4 x0 = lds128(rbase + 16 * ((2 * c) ^ sw));
    const uint4 x1 = lds128(rbase + 16 * ((2 * c + 1) ^ sw));
    const uint32_t b8[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    const uint32_t iw[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const uint32_t id = (iw[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
      if (mkey != 0xFFFFFFFFu && b8[q] == mkey) mid = min(mid, id);
      if (id == p.ell) {
        mine.lcode = ok_bits(b8[q]) ? 2u : 1u;
        mine.l_bits = b8[q];
      }
    }
  }
  mine.min_bid = mid;
}

__device__ __forceinline__ void emit_group(const RP& p, uint64_t gl, bool active, const GroupAcc& mine,
                                           ThreadAcc& t, uint64_t* sh_c, uint32_t* sh_perf,
                                           uint32_t* sh_gain, uint32_t* sh_bb) {
  if (p.mode == MODE_FUSED) {
    finalize_lane(p, gl, active, mine, t, sh_c, sh_perf, sh_gain, sh_bb);
  } else if (active) {  // MODE_GROUP_PARTIALS: per-group values for the NCCL MIN/MAX/SUM merge
    p.g_key[gl] = mine.min_bits == 0xFFFFFFFFu ? ~0ull : (((uint64_t)mine.min_bits << 32) | mine.min_bid);
    p.g_lcode[gl] = mine.lcode == 2 ? ((1ull << 32) | mine.l_bits) : (uint64_t)mine.lcode;
    p.g_cnt[3 * gl + 0] = mine.n_ok;
    p.g_cnt[3 * gl + 1] = mine.n_nan;
    p.g_cnt[3 * gl + 2] = mine.n_rows;
  }
}

// a6/a7 for tables of uniform 32-row groups with 16-byte aligned arrays (BASELINE configs[4]):
// each warp streams its batches of 32 groups through a cp.async stage; as soon as lane j has
// folded group j the next batch is requested, so its loads fly while the batch is finalised.
__global__ void __launch_bounds__(kThreads, 3) reduce_uniform32_kernel(RP p) {
  extern __shared__ uint64_t dyn[];
  uint64_t* sh_c = dyn;
  uint32_t* sh = reinterpret_cast<uint32_t*>(dyn + kNC);
  uint32_t* sh_perf = sh;
  uint32_t* sh_gain = sh + (p.nb + 1);
  uint32_t* sh_bb = sh_gain + (p.cap * p.nb + 1);
  uint8_t* stage = reinterpret_cast<uint8_t*>(dyn) + kNC * 8 + ((p.smem_words * 4 + 15) & ~15u);
  ThreadAcc t;
  init_shared(p, sh_c, sh, t);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // one stage per warp: [runtimes 4 KB | ids 2 KB]
  uint8_t* wstage = stage + (size_t)wib * (1024 * 4 + 1024 * 2);
  auto D = [&](int b) { return reinterpret_cast<float4*>(wstage + b * (1024 * 4 + 1024 * 2)); };
  auto DI = [&](int b) { return reinterpret_cast<uint4*>(wstage + b * (1024 * 4 + 1024 * 2) + 1024 * 4); };
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  // batches of 32 complete 32-row groups: a short last group (n_rows < 32 G) always goes to
  // the tail below, which bounds its rows by n_rows
  const uint64_t full_batches = (p.n_rows / 32) / 32;
  uint64_t bi = warp;
  if (bi < full_batches) uniform_prefetch(p, bi * 32, D(0), DI(0), lane);
  for (; bi < full_batches; bi += nwarps) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    GroupAcc mine;
    acc_init(mine);
    uniform_fold(p, (uint32_t)__cvta_generic_to_shared(D(0)), (uint32_t)__cvta_generic_to_shared(DI(0)), lane, mine);
    __syncwarp();
    // the stage is free again: the next batch streams in while this one is finalised
    const uint64_t nxt = bi + nwarps;
    if (nxt < full_batches) uniform_prefetch(p, nxt * 32, D(0), DI(0), lane);
    emit_group(p, bi * 32 + lane, true, mine, t, sh_c, sh_perf, sh_gain, sh_bb);
  }
  // tail: the last < 32 groups (the last one possibly short), warp-per-group folding
  const uint64_t tail0 = full_batches * 32;
  if (tail0 < p.n_groups && warp == (full_batches % nwarps)) {
    const int nj = (int)(p.n_groups - tail0);
    GroupAcc mine;
    acc_init(mine);
    for (int j = 0; j < nj; j++) {
      const int64_t r0 = (int64_t)(tail0 + j) * 32;
      const int64_t r1 = min(r0 + 32, (int64_t)p.n_rows);
      GroupAcc a;
      acc_init(a);
      const int64_t r = r0 + lane;
      const bool v = r < r1;
      fold_chunk(a, v, v ? __float_as_uint(__ldcs(p.rt + r)) : 0u, v ? (uint32_t)__ldcs(p.bid + r) : 0u, p.ell);
      if (lane == j) mine = a;
    }
    emit_group(p, tail0 + lane, lane < nj, mine, t, sh_c, sh_perf, sh_gain, sh_bb);
  }
  (void)FULL;
  flush(p, t, sh_c, sh);
}

// a6/a7: a warp takes 32 consecutive groups.  When every group has <= 32 rows and the batch
// has <= 1024 rows (always, for the paper's tables), the rows are loaded with coalesced loads
// (8 in flight per lane) into the warp's shared-memory stage and lane j then folds group j's
// rows sequentially; otherwise the warp folds each group with redux/ballot (fallback).
__global__ void __launch_bounds__(kThreads, 2) reduce_groups_kernel(RP p) {
  extern __shared__ uint64_t dyn[];
  uint64_t* sh_c = dyn;
  uint32_t* sh = reinterpret_cast<uint32_t*>(dyn + kNC);
  uint32_t* sh_perf = sh;
  uint32_t* sh_gain = sh + (p.nb + 1);
  uint32_t* sh_bb = sh_gain + (p.cap * p.nb + 1);
  uint8_t* stage = reinterpret_cast<uint8_t*>(dyn) + kNC * 8 + ((p.smem_words * 4 + 15) & ~15u);
  ThreadAcc t;
  init_shared(p, sh_c, sh, t);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* s_rt = reinterpret_cast<uint32_t*>(stage) + (size_t)wib * kStagePad;
  uint16_t* s_id = reinterpret_cast<uint16_t*>(stage + (size_t)kWarps * kStagePad * 4) + (size_t)wib * kStagePad;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = warp * 32; base < p.n_groups; base += nwarps * 32) {
    const int nj = (int)min((uint64_t)32, p.n_groups - base);
    const uint64_t gl = base + lane;
    int64_t lo = 0, hi = 0;
    if (lane < nj) {
      if (p.rpg) {
        lo = (int64_t)(gl * p.rpg);
        hi = min((int64_t)(lo + p.rpg), (int64_t)p.n_rows);
      } else {
        lo = p.off[gl];
        hi = p.off[gl + 1];
      }
    }
    const int64_t R0 = __shfl_sync(FULL, lo, 0);
    const int64_t R1 = __shfl_sync(FULL, hi, nj - 1);
    const uint32_t maxlen = __reduce_max_sync(FULL, (uint32_t)(hi - lo));
    const int64_t total = R1 - R0;
    GroupAcc mine;
    acc_init(mine);
    const uint32_t minlen = __reduce_min_sync(FULL, lane < nj ? (uint32_t)(hi - lo) : 32u);
    if (nj == 32 && maxlen == 32 && minlen == 32 && p.vec && (R0 & 7) == 0) {
      // a batch of 32 full 32-row groups (configs[2]/[3] apart from the last group): the
      // uniform tables' swizzled cp.async stage and one-pass fold, in this warp's stage
      float4* d = reinterpret_cast<float4*>(s_rt);
      uint4* di = reinterpret_cast<uint4*>(s_id);
      uniform_prefetch_rows(p, (uint64_t)R0, d, di, lane);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      uniform_fold(p, (uint32_t)__cvta_generic_to_shared(d), (uint32_t)__cvta_generic_to_shared(di), lane, mine);
      __syncwarp();
    } else if (maxlen <= 32 && total >= 0 && total <= kStageRows) {
      const int tot = (int)total;
      constexpr int kU = 16;  // rows in flight per lane
      for (int r0 = 0; r0 < tot; r0 += 32 * kU) {
        uint32_t v[kU];
        uint16_t b[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
          const int r = r0 + u * 32 + lane;
          v[u] = r < tot ? __float_as_uint(__ldcs(p.rt + R0 + r)) : 0u;
          b[u] = r < tot ? __ldcs(p.bid + R0 + r) : (uint16_t)0;
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
          const int r = r0 + u * 32 + lane;
          if (r < tot) {
            s_rt[r + (r >> 5)] = v[u];
            s_id[r + (r >> 5)] = b[u];
          }
        }
      }
      __syncwarp();
      if (lane < nj) {
        const int a1 = (int)(hi - R0);
        for (int r = (int)(lo - R0); r < a1; r++) fold_row(mine, s_rt[r + (r >> 5)], s_id[r + (r >> 5)], p.ell);
      }
      __syncwarp();
    } else {
      for (int j = 0; j < nj; j++) {
        const int64_t r0 = __shfl_sync(FULL, lo, j), r1 = __shfl_sync(FULL, hi, j);
        GroupAcc a;
        acc_init(a);
        for (int64_t c = r0; c < r1; c += 32) {
          const int64_t r = c + lane;
          const bool v = r < r1;
          fold_chunk(a, v, v ? __float_as_uint(__ldcs(p.rt + r)) : 0u, v ? (uint32_t)__ldcs(p.bid + r) : 0u, p.ell);
        }
        if (lane == j) mine = a;
      }
    }
    if (p.mode == MODE_FUSED) {
      finalize_lane(p, gl, lane < nj, mine, t, sh_c, sh_perf, sh_gain, sh_bb);
    } else if (lane < nj) {  // MODE_GROUP_PARTIALS: per-group values for the NCCL MIN/MAX/SUM merge
      p.g_key[gl] = mine.min_bits == 0xFFFFFFFFu ? ~0ull : (((uint64_t)mine.min_bits << 32) | mine.min_bid);
      p.g_lcode[gl] = mine.lcode == 2 ? ((1ull << 32) | mine.l_bits) : (uint64_t)mine.lcode;
      p.g_cnt[3 * gl + 0] = mine.n_ok;
      p.g_cnt[3 * gl + 1] = mine.n_nan;
      p.g_cnt[3 * gl + 2] = mine.n_rows;
    }
  }
  flush(p, t, sh_c, sh);
}

__global__ void __launch_bounds__(kThreads) finalize_merged_kernel(RP p) {
  extern __shared__ uint64_t dyn[];
  uint64_t* sh_c = dyn;
  uint32_t* sh = reinterpret_cast<uint32_t*>(dyn + kNC);
  uint32_t* sh_perf = sh;
  uint32_t* sh_gain = sh + (p.nb + 1);
  uint32_t* sh_bb = sh_gain + (p.cap * p.nb + 1);
  ThreadAcc t;
  init_shared(p, sh_c, sh, t);
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = warp * 32; base < p.n_groups; base += nwarps * 32) {
    const uint64_t g = base + lane;
    const bool active = g < p.n_groups;
    GroupAcc a;
    acc_init(a);
    if (active) {
      const uint64_t key = p.g_key[g], lc = p.g_lcode[g];
      a.min_bits = key == ~0ull ? 0xFFFFFFFFu : (uint32_t)(key >> 32);
      a.min_bid = key == ~0ull ? 0xFFFFFFFFu : (uint32_t)(key & 0xFFFFFFFFu);
      a.n_ok = p.g_cnt[3 * g];
      a.n_nan = p.g_cnt[3 * g + 1];
      a.n_rows = p.g_cnt[3 * g + 2];
      a.lcode = lc >> 32 ? 2u : (uint32_t)lc;
      a.l_bits = (uint32_t)(lc & 0xFFFFFFFFu);
    }
    finalize_lane(p, g, active, a, t, sh_c, sh_perf, sh_gain, sh_bb);
  }
  flush(p, t, sh_c, sh);
}


// Zero the partial vector and reset the key min/max in one launch (was a memset + a kernel).
__global__ void init_partials(uint64_t* __restrict__ partials, size_t plen, uint64_t* __restrict__ mm) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < plen; i += (size_t)gridDim.x * blockDim.x)
    partials[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    mm[0] = ~0ull; mm[1] = 0; mm[2] = ~0ull; mm[3] = 0;
  }
}

size_t partials_len(const lscat_reduce_opts& o) {
  return (size_t)kNC + (o.bins_per_unit + 1) + ((size_t)o.gain_cap * o.bins_per_unit + 1) +
         (size_t)o.n_matrices * o.n_blocks * (o.block_profile ? 3 : 1) +
         (o.kernel_rollup ? (size_t)8 + o.bins_per_unit + 1 : 0);
}

// Block profile (Figs. 2/4; reading R-22): a second pass over this rank's rows once
// every group's best runtime is final (after the a9 per-group merge when point-sharded).
// Warp per group, lanes over rows; per ok row of a defined group the performance best / r_b
// as floor(RN(best / r_b) * 2^31) is added to a shared (matrix, block) slot; one flush per CTA.
__global__ void __launch_bounds__(256) profile_kernel(RP p, const float* __restrict__ best_rt,
                                                      const uint32_t* __restrict__ gflags,
                                                      uint64_t* __restrict__ prof_sum,
                                                      uint64_t* __restrict__ prof_cnt) {
  extern __shared__ uint64_t sp[];
  const uint32_t ML = p.M * p.L;
  uint64_t* s_sum = sp;
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(sp + ML);
  for (uint32_t i = threadIdx.x; i < ML; i += blockDim.x) { s_sum[i] = 0; s_cnt[i] = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g = warp; g < p.n_groups; g += nwarps) {
    if (!(gflags[g] & LSCAT_GF_DEFINED)) continue;
    const double b = (double)best_rt[g];
    const uint32_t mat = p.gmat ? p.gmat[g] : (uint32_t)((p.first_group + g) % p.M);
    int64_t r0, r1;
    if (p.rpg) {
      r0 = (int64_t)(g * p.rpg);
      r1 = min(r0 + (int64_t)p.rpg, (int64_t)p.n_rows);
    } else {
      r0 = p.off[g];
      r1 = p.off[g + 1];
    }
    for (int64_t r = r0 + lane; r < r1; r += 32) {
      const float v = __ldcs(p.rt + r);
      if (!ok_bits(__float_as_uint(v))) continue;
      const uint32_t id = __ldcs(p.bid + r);
      if (id >= p.L || mat >= p.M) continue;  // counted as LSCAT_P_BAD_IDS by the reducer
      const uint64_t q = (uint64_t)__dmul_rn(__ddiv_rn(b, (double)v), 2147483648.0);
      atomicAdd((unsigned long long*)&s_sum[mat * p.L + id], (unsigned long long)q);
      atomicAdd(&s_cnt[mat * p.L + id], 1u);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < ML; i += blockDim.x) {
    if (s_cnt[i]) {
      atomicAdd((unsigned long long*)&prof_sum[i], (unsigned long long)s_sum[i]);
      atomicAdd((unsigned long long*)&prof_cnt[i], (unsigned long long)s_cnt[i]);
    }
  }
}

// ---- per-kernel roll-up (R-26) ------------------------------------------
// Over the groups [lo, hi) this rank accumulated, a thread at each kernel's first group folds
// the kernel's records (c = ratio-defined groups, S = sum of floor(perf 2^52) as a 128-bit
// integer, any best block != l).  Kernels wholly inside (lo, hi) are finalised here; the
// segment touching lo and the one touching hi may continue on another rank, so they go to two
// boundary records (kernel id + partial sums) that rank 0 merges after an all-gather.
constexpr int kRollupWords = 8;   // counters region of the roll-up partials
constexpr int kBndWords = 5;      // boundary record: kid | 1 << 32, c, S lo64, S hi64, not_best

struct RollupArgs {
  const uint64_t* krec;
  const uint32_t* gkern;  // NULL -> (first_group + g) / M
  uint64_t first_group, lo, hi;
  uint32_t M, nb, pln, pld, bln, bld;
  int mshift;             // log2(M) when M is a power of two, else -1
  uint64_t* part;         // roll-up region of the partial vector: [8] counters, [nb+1] hist
  uint64_t* bnd;          // [2 * kBndWords] this rank's boundary records
};

__device__ __forceinline__ uint32_t kid_of(const RollupArgs& q, uint64_t g) {
  if (q.gkern) return q.gkern[g];
  const uint64_t ag = q.first_group + g;  // implicit: a shift when M is a power of two
  if (q.mshift >= 0) return (uint32_t)(ag >> q.mshift);
  if (ag < (1ull << 32)) return (uint32_t)ag / q.M;
  return (uint32_t)(ag / q.M);
}

// Per-thread roll-up counters (flushed once per warp: the per-kernel increments all go to the
// same six words, so per-kernel atomics would serialise).
struct KAcc {
  unsigned long long v[6];  // n_kernels, not_best, perf_lt, band, mean fx hi, mean fx lo
};

// One kernel's roll-up (exact: 128-bit products of the fixed-point sum, R-26).
__device__ void kernel_fin(const RollupArgs& q, uint64_t c, unsigned __int128 S, bool not_best,
                           KAcc& a, uint32_t* hist32, unsigned long long* hist64) {
  if (c == 0) return;
  const unsigned __int128 cd = (unsigned __int128)c << 52;  // kernel-mean perf = S / cd
  const bool lt = (unsigned __int128)q.pld * S < (unsigned __int128)q.pln * cd;
  const bool band = lt && (unsigned __int128)q.bld * S >= (unsigned __int128)q.bln * cd;
  // 128-bit divisions are long software sequences: estimate in double, then fix up exactly
  // with 128-bit products (the same integers as a division would give)
  const unsigned __int128 nbS = (unsigned __int128)q.nb * S;
  const double sd = (double)(uint64_t)S + (double)(uint64_t)(S >> 64) * 0x1p64;
  int64_t bin = (int64_t)(sd / (double)c * (double)q.nb * 0x1p-52);  // largest j: j cd <= nb S
  if (bin < 0) bin = 0;
  while (bin < (int64_t)q.nb && (unsigned __int128)(bin + 1) * cd <= nbS) bin++;
  while (bin > 0 && (unsigned __int128)bin * cd > nbS) bin--;
  uint64_t kfx = (uint64_t)(sd / (double)c);  // floor(S / c) <= 2^52
  while ((unsigned __int128)(kfx + 1) * c <= S) kfx++;
  while (kfx > 0 && (unsigned __int128)kfx * c > S) kfx--;
  a.v[0] += 1;
  a.v[1] += not_best;
  a.v[2] += lt;
  a.v[3] += band;
  a.v[4] += kfx >> 21;
  a.v[5] += kfx & ((1ull << 21) - 1);
  if (hist32) atomicAdd(&hist32[bin], 1u);
  else atomicAdd(&hist64[bin], 1ull);
}

// multiply-high reciprocals m_c = floor((2^64 - 1) / c) + 1 of c = 2..32 (m_0, m_1 unused)
__constant__ uint64_t kRcp32[33] = {
    0x0000000000000000ull, 0x0000000000000000ull, 0x8000000000000000ull,
    0x5555555555555556ull, 0x4000000000000000ull, 0x3333333333333334ull,
    0x2aaaaaaaaaaaaaabull, 0x2492492492492493ull, 0x2000000000000000ull,
    0x1c71c71c71c71c72ull, 0x199999999999999aull, 0x1745d1745d1745d2ull,
    0x1555555555555556ull, 0x13b13b13b13b13b2ull, 0x124924924924924aull,
    0x1111111111111112ull, 0x1000000000000000ull, 0x0f0f0f0f0f0f0f10ull,
    0x0e38e38e38e38e39ull, 0x0d79435e50d79436ull, 0x0ccccccccccccccdull,
    0x0c30c30c30c30c31ull, 0x0ba2e8ba2e8ba2e9ull, 0x0b21642c8590b217ull,
    0x0aaaaaaaaaaaaaabull, 0x0a3d70a3d70a3d71ull, 0x09d89d89d89d89d9ull,
    0x097b425ed097b426ull, 0x0924924924924925ull, 0x08d3dcb08d3dcb09ull,
    0x0888888888888889ull, 0x0842108421084211ull, 0x0800000000000000ull,
};

// kernel_fin for kernels of <= 32 groups (S <= c 2^52 <= 2^57): the same integers with 64-bit
// arithmetic and 64 x 64 -> 128-bit products by mul.hi (no 128-bit multiplies or f64 division).
__device__ __forceinline__ bool mul_lt(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {  // a b < c d
  const uint64_t h1 = __umul64hi(a, b), h2 = __umul64hi(c, d);
  return h1 < h2 || (h1 == h2 && a * b < c * d);
}
__device__ void kernel_fin_small(const RollupArgs& q, uint32_t c, uint64_t S, bool not_best, KAcc& a,
                                 uint32_t* hist32) {
  if (c == 0) return;
  const uint64_t cd = (uint64_t)c << 52;  // kernel-mean perf = S / cd
  const bool lt = mul_lt(q.pld, S, q.pln, cd);
  const bool band = lt && !mul_lt(q.bld, S, q.bln, cd);
  // divisions by c <= 32 as a multiply-high by m = floor((2^64 - 1) / c) + 1 (c > 1), then one
  // exact fix-up step each way (64-bit integer division is a long software sequence)
  const uint64_t m = kRcp32[c];
  auto divc = [&](uint64_t x) -> uint64_t {
    if (c == 1) return x;
    uint64_t d = __umul64hi(x, m);
    if (d * c > x) d--;
    if ((d + 1) * c <= x) d++;
    return d;
  };
  // bin = floor(nb S / cd) = floor(floor(nb S / 2^52) / c)
  const uint64_t nbS_lo = (uint64_t)q.nb * S, nbS_hi = __umul64hi((uint64_t)q.nb, S);
  uint64_t bin = divc((nbS_hi << 12) | (nbS_lo >> 52));
  if (bin > q.nb) bin = q.nb;  // perf <= 1 (defensive: the histogram has nb + 1 bins)
  const uint64_t kfx = divc(S);  // floor(S / c) <= 2^52
  a.v[0] += 1;
  a.v[1] += not_best;
  a.v[2] += lt;
  a.v[3] += band;
  a.v[4] += kfx >> 21;
  a.v[5] += kfx & ((1ull << 21) - 1);
  atomicAdd(&hist32[bin], 1u);
}

__device__ __forceinline__ void write_bnd(const RollupArgs& q, int slot, uint32_t k, uint64_t c,
                                          unsigned __int128 S, bool nbst) {
  uint64_t* b = q.bnd + slot * kBndWords;
  b[0] = (uint64_t)k | (1ull << 32);
  b[1] = c;
  b[2] = (uint64_t)S;
  b[3] = (uint64_t)(S >> 64);
  b[4] = nbst;
}

// Warp-cooperative: a warp takes a contiguous range of 32-group chunks, lane j holds group
// base + j; kernels are the runs of equal kernel ids (segments), summed with a segmented scan
// (plain inclusive scans minus the value before each segment's head).  A segment ending
// inside the chunk is finalised by its last lane; the one reaching lane 31 is carried to the
// next chunk.  A warp skips the leading groups of a kernel that began before its range (the
// previous warp finishes it) and reads past its range end to finish its last kernel.
__global__ void __launch_bounds__(256) rollup_kernel(RollupArgs q) {
  extern __shared__ unsigned long long rs[];
  unsigned long long* cnt = rs;                                  // [kRollupWords]
  uint32_t* hist = reinterpret_cast<uint32_t*>(rs + kRollupWords);  // [nb + 1]
  for (uint32_t i = threadIdx.x; i < kRollupWords; i += blockDim.x) cnt[i] = 0;
  for (uint32_t i = threadIdx.x; i <= q.nb; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  KAcc acc{};
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint64_t nch = (q.hi - q.lo + 31) / 32;
  const uint64_t Wt = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t ch0 = w * nch / Wt, ch1 = (w + 1) * nch / Wt;
  if (ch0 < ch1) {
    const uint64_t g_begin = q.lo + ch0 * 32, g_end = min(q.lo + ch1 * 32, q.hi);
    bool skipping = g_begin > q.lo;
    const uint32_t skip_k = skipping ? kid_of(q, g_begin - 1) : 0u;
    bool cv = false, cfirst = false;  // carried kernel (warp-uniform)
    uint32_t ck = 0;
    uint64_t cc = 0, cn = 0;
    unsigned __int128 cS = 0;
    for (uint64_t base = g_begin; base < q.hi; base += 32) {
      const bool beyond = base >= g_end;
      if (beyond && !cv) break;
      const uint64_t g = base + lane;
      const bool in = g < q.hi;
      const uint32_t k = in ? kid_of(q, g) : 0u;
      const uint64_t r = in ? q.krec[g] : 0ull;
      bool inc = in;
      if (skipping) {
        const bool sk = in && k == skip_k;
        inc = inc && !sk;
        skipping = __all_sync(FULL, sk || !in) && __any_sync(FULL, in) && base + 32 < q.hi;
      }
      if (beyond) inc = inc && k == ck;  // only the carried kernel's continuation
      const uint64_t vc = (inc && ((r >> 53) & 1)) ? 1ull : 0ull;
      const uint64_t vs = vc ? (r & ((1ull << 53) - 1)) : 0ull;
      const uint64_t vn = vc ? ((r >> 54) & 1) : 0ull;
      const uint32_t pk = __shfl_up_sync(FULL, k, 1);
      const bool pin = __shfl_up_sync(FULL, inc, 1);
      const bool head = lane == 0 || k != pk || inc != pin;
      const unsigned hm = __ballot_sync(FULL, head);
      uint64_t ic = vc, is = vs, in_ = vn;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t yc = __shfl_up_sync(FULL, ic, o), ys = __shfl_up_sync(FULL, is, o),
                       yn = __shfl_up_sync(FULL, in_, o);
        if (lane >= o) { ic += yc; is += ys; in_ += yn; }
      }
      const int start = 31 - __clz(hm & (FULL >> (31 - lane)));
      const int src = start ? start - 1 : 0;
      uint64_t bc = __shfl_sync(FULL, ic, src), bs = __shfl_sync(FULL, is, src), bn = __shfl_sync(FULL, in_, src);
      if (start == 0) bc = bs = bn = 0;
      const bool tail = lane == 31 || ((hm >> (lane + 1)) & 1);
      const bool l0_in = __shfl_sync(FULL, inc, 0);
      const uint32_t l0_k = __shfl_sync(FULL, k, 0);
      const bool cont = cv && l0_in && l0_k == ck;  // the carried kernel continues at lane 0
      if (cv && !cont && lane == 0) {               // it ended exactly at the chunk boundary
        if (cfirst) write_bnd(q, 0, ck, cc, cS, cn != 0);
        else kernel_fin(q, cc, cS, cn != 0, acc, hist, nullptr);
      }
      uint64_t tc = ic - bc, tn = in_ - bn;
      unsigned __int128 tS = is - bs;
      bool tfirst = base + start == q.lo;
      if (start == 0 && cont) { tc += cc; tS += cS; tn += cn; tfirst = cfirst; }
      if (tail && inc && lane != 31) {               // a kernel that ends inside this chunk
        if (tfirst || g + 1 == q.hi) write_bnd(q, tfirst ? 0 : 1, k, tc, tS, tn != 0);  // rank edges
        else kernel_fin(q, tc, tS, tn != 0, acc, hist, nullptr);
      }
      // carry = lane 31's segment when it is included (it may continue in the next chunk)
      cv = __shfl_sync(FULL, inc, 31);
      ck = __shfl_sync(FULL, k, 31);
      cc = __shfl_sync(FULL, tc, 31);
      cn = __shfl_sync(FULL, tn, 31);
      const uint64_t slo = __shfl_sync(FULL, (uint64_t)tS, 31), shi = __shfl_sync(FULL, (uint64_t)(tS >> 64), 31);
      cS = ((unsigned __int128)shi << 64) | slo;
      cfirst = __shfl_sync(FULL, tfirst, 31);
    }
    if (cv && lane == 0) {  // the last kernel reaches hi: it may continue on the next rank
      write_bnd(q, cfirst ? 0 : 1, ck, cc, cS, cn != 0);
    }
  }
#pragma unroll
  for (int i = 0; i < 6; i++) {
    unsigned long long x = acc.v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&cnt[i], x);
  }
  __syncthreads();
  unsigned long long* gc = reinterpret_cast<unsigned long long*>(q.part);
  for (uint32_t i = threadIdx.x; i < kRollupWords; i += blockDim.x)
    if (cnt[i]) atomicAdd(&gc[i], cnt[i]);
  for (uint32_t i = threadIdx.x; i <= q.nb; i += blockDim.x)
    if (hist[i]) atomicAdd(&gc[kRollupWords + i], (unsigned long long)hist[i]);
}

// Implicit kernel ids with a power-of-two M <= 32 (configs[4]): lane j of a warp takes
// kernel k = kb + j whole (its M records read sequentially: a warp reads 32 M contiguous
// records), sums c, S (< 2^58) and the not-best flag in registers and finalises the kernel, or
// writes the boundary record when the kernel reaches past this rank's range (it may continue on
// a neighbouring rank).  Same totals as rollup_kernel, with every lane finalising a kernel.
__global__ void __launch_bounds__(256) rollup_uniform_kernel(RollupArgs q) {
  extern __shared__ unsigned long long rs[];
  unsigned long long* cnt = rs;                                  // [kRollupWords]
  uint32_t* hist = reinterpret_cast<uint32_t*>(rs + kRollupWords);  // [nb + 1]
  for (uint32_t i = threadIdx.x; i < kRollupWords; i += blockDim.x) cnt[i] = 0;
  for (uint32_t i = threadIdx.x; i <= q.nb; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  KAcc acc{};
  const uint32_t M = q.M;
  const uint64_t alo = q.first_group + q.lo, ahi = q.first_group + q.hi;  // absolute range
  const uint64_t k0 = alo >> q.mshift, k1 = (ahi + M - 1) >> q.mshift;   // kernels touched
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = k0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < k1; k += T) {
    const uint64_t g0 = k << q.mshift;  // the kernel's first absolute group
    uint32_t c = 0, nbst = 0;
    uint64_t S = 0;
    for (uint32_t i = 0; i < M; i++) {
      const uint64_t ga = g0 + i;
      const uint64_t r = (ga >= alo && ga < ahi) ? q.krec[ga - q.first_group] : 0ull;
      const uint32_t rd = (uint32_t)((r >> 53) & 1);
      c += rd;
      S += rd ? (r & ((1ull << 53) - 1)) : 0ull;
      nbst |= rd & (uint32_t)((r >> 54) & 1);
    }
    if (g0 >= alo && g0 + M <= ahi) kernel_fin_small(q, c, S, nbst != 0, acc, hist);
    else write_bnd(q, g0 < alo ? 0 : 1, (uint32_t)k, c, (unsigned __int128)S, nbst != 0);
  }
#pragma unroll
  for (int i = 0; i < 6; i++) {
    unsigned long long x = acc.v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&cnt[i], x);
  }
  __syncthreads();
  unsigned long long* gc = reinterpret_cast<unsigned long long*>(q.part);
  for (uint32_t i = threadIdx.x; i < kRollupWords; i += blockDim.x)
    if (cnt[i]) atomicAdd(&gc[i], cnt[i]);
  for (uint32_t i = threadIdx.x; i <= q.nb; i += blockDim.x)
    if (hist[i]) atomicAdd(&gc[kRollupWords + i], (unsigned long long)hist[i]);
}

// Rank 0 merges every rank's two boundary records in rank order (equal kernel ids are adjacent
// because a kernel's groups are contiguous) and finalises the merged kernels.
__global__ void rollup_boundary_kernel(RollupArgs q, const uint64_t* __restrict__ all, int nrec) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long* gc = reinterpret_cast<unsigned long long*>(q.part);
  KAcc acc{};
  bool have = false;
  uint32_t kid = 0;
  uint64_t c = 0;
  unsigned __int128 S = 0;
  bool nbst = false;
  for (int i = 0; i < nrec; i++) {
    const uint64_t* b = all + (size_t)i * kBndWords;
    if (!(b[0] >> 32)) continue;
    const uint32_t k = (uint32_t)b[0];
    if (have && k != kid) {
      kernel_fin(q, c, S, nbst, acc, nullptr, gc + kRollupWords);
      have = false;
    }
    if (!have) { have = true; kid = k; c = 0; S = 0; nbst = false; }
    c += b[1];
    S += ((unsigned __int128)b[3] << 64) | b[2];
    nbst |= b[4] != 0;
  }
  if (have) kernel_fin(q, c, S, nbst, acc, nullptr, gc + kRollupWords);
  for (int i = 0; i < 6; i++) gc[i] += acc.v[i];
}

bool opts_ok(const lscat_reduce_opts* o) {
  if (!o) return false;
  if (o->n_blocks == 0 || o->n_blocks > 65535 || o->largest_block_id >= o->n_blocks) return false;
  if (o->n_matrices == 0 || o->bins_per_unit == 0 || o->gain_cap == 0) return false;
  if (o->bins_per_unit > 100000 || (uint64_t)o->gain_cap * o->bins_per_unit > 1000000) return false;
  if (o->gain_gt_den == 0 || o->perf_lt_den == 0 || o->band_lo_den == 0) return false;
  if ((uint64_t)o->gain_gt_den + o->gain_gt_num >= (1u << 29)) return false;
  if (o->perf_lt_num >= (1u << 29) || o->perf_lt_den >= (1u << 29)) return false;
  if (o->band_lo_num >= (1u << 29) || o->band_lo_den >= (1u << 29)) return false;
  if (o->nan_policy > LSCAT_COMPLETE_ONLY) return false;
  if (o->block_profile && (uint64_t)o->n_matrices * o->n_blocks * 12 > 200 * 1024) return false;
  if (o->kernel_rollup > 1 || o->block_profile > 1) return false;
  if (o->n_percentiles > 64 || (o->n_percentiles && !o->percentiles)) return false;
  for (uint32_t i = 0; i < o->n_percentiles; i++)
    if (!(o->percentiles[i] >= 0.0 && o->percentiles[i] <= 1.0)) return false;
  return true;
}


}  // namespace
}  // namespace lscat

using namespace lscat;

extern "C" {

void lscat_reduce_opts_default(lscat_reduce_opts* o, uint32_t n_blocks, uint32_t n_matrices) {
  if (!o) return;
  memset(o, 0, sizeof *o);
  o->n_blocks = n_blocks;
  o->largest_block_id = n_blocks ? n_blocks - 1 : 0;
  o->n_matrices = n_matrices;
  o->nan_policy = LSCAT_SKIPNA;
  o->bins_per_unit = 100;
  o->gain_cap = 10;
  o->gain_gt_num = 1; o->gain_gt_den = 5;
  o->perf_lt_num = 17; o->perf_lt_den = 20;
  o->band_lo_num = 2; o->band_lo_den = 5;
  o->point_sharded = 0;
  o->keep_values = 1;
}

size_t lscat_partials_len(const lscat_reduce_opts* o) { return opts_ok(o) ? partials_len(*o) : 0; }

static lscat_status reduce_enqueue(lscat_ctx* ctx, const lscat_table* T, const lscat_reduce_opts* o,
                                   lscat_reduce_out* out, void* stream) {
  LSCAT_CHECK_CTX(ctx);
  if (!T || !opts_ok(o)) return fail(ctx, LSCAT_ERR_INVALID_ARG, "reduce_table: bad table or options");
  if (!T->runtime_ms || !T->block_id || (!T->rows_per_group && !T->group_offset) ||
      T->mem > LSCAT_MEM_HOST)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "reduce_table: table needs runtime_ms, block_id and offsets");
  if (T->rows_per_group && (T->n_groups != (T->n_rows + T->rows_per_group - 1) / T->rows_per_group))
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "reduce_table: n_groups != ceil(n_rows / rows_per_group)");
  const size_t sh_words = (o->bins_per_unit + 1) + ((size_t)o->gain_cap * o->bins_per_unit + 1) +
                          (size_t)o->n_matrices * o->n_blocks;
  const size_t smem_fin = kNC * 8 + sh_words * 4;
  const size_t smem_hist = kNC * 8 + ((sh_words * 4 + 15) & ~(size_t)15);
  size_t smem = smem_hist + kStageBytes;
  if (smem > 200 * 1024)
    return fail(ctx, LSCAT_ERR_UNSUPPORTED, "reduce_table: histograms need %zu B of shared memory", smem);
  cudaStream_t s = (cudaStream_t)stream;
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));
  const uint64_t G = T->n_groups, n = T->n_rows;
  lscat_reduce_out dummy{};
  if (!out) out = &dummy;
  cudaError_t err;

  RP p{};
  const uint32_t* gkern = T->group_kernel;
  // stage host tables through device scratch (e2e path)
  if (T->mem == LSCAT_MEM_HOST) {
    float* rt = (float*)scratch(ctx, "h_rt", n * 4, &err);
    if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
    uint16_t* bid = (uint16_t*)scratch(ctx, "h_bid", n * 2, &err);
    if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
    LSCAT_CUDA(ctx, cudaMemcpyAsync(rt, T->runtime_ms, n * 4, cudaMemcpyHostToDevice, s));
    LSCAT_CUDA(ctx, cudaMemcpyAsync(bid, T->block_id, n * 2, cudaMemcpyHostToDevice, s));
    p.rt = rt;
    p.bid = bid;
    if (!T->rows_per_group) {
      int64_t* off = (int64_t*)scratch(ctx, "h_off", (G + 1) * 8, &err);
      if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
      LSCAT_CUDA(ctx, cudaMemcpyAsync(off, T->group_offset, (G + 1) * 8, cudaMemcpyHostToDevice, s));
      p.off = off;
    }
    if (T->group_matrix) {
      uint32_t* gm = (uint32_t*)scratch(ctx, "h_gm", G * 4, &err);
      if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
      LSCAT_CUDA(ctx, cudaMemcpyAsync(gm, T->group_matrix, G * 4, cudaMemcpyHostToDevice, s));
      p.gmat = gm;
    }
    if (T->group_kernel && o->kernel_rollup) {
      uint32_t* gk = (uint32_t*)scratch(ctx, "h_gk", G * 4, &err);
      if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
      LSCAT_CUDA(ctx, cudaMemcpyAsync(gk, T->group_kernel, G * 4, cudaMemcpyHostToDevice, s));
      gkern = gk;
    }
  } else {
    p.rt = T->runtime_ms;
    p.bid = T->block_id;
    p.off = T->group_offset;
    p.gmat = T->group_matrix;
  }
  p.vec = ((uintptr_t)p.rt % 16 == 0) && ((uintptr_t)p.bid % 16 == 0);
  p.n_groups = G;
  p.first_group = T->first_group;
  p.rpg = T->rows_per_group;
  p.n_rows = n;
  p.L = o->n_blocks; p.ell = o->largest_block_id; p.M = o->n_matrices; p.policy = o->nan_policy;
  p.nb = o->bins_per_unit; p.cap = o->gain_cap;
  p.ggn = o->gain_gt_num; p.ggd = o->gain_gt_den; p.pln = o->perf_lt_num; p.pld = o->perf_lt_den;
  p.bln = o->band_lo_num; p.bld = o->band_lo_den;
  p.smem_words = (uint32_t)sh_words;
  p.o_best = out->best_block_id;
  p.o_bestrt = out->best_runtime;
  p.o_perf = out->perf;
  p.o_gain = out->gain;
  p.o_flags = out->flags;
  if (o->block_profile) {
    if (!p.o_bestrt) { p.o_bestrt = (float*)scratch(ctx, "bestrt", G * 4, &err); if (err) return cuda_fail(ctx, err, "scratch"); }
    if (!p.o_flags) { p.o_flags = (uint32_t*)scratch(ctx, "gflags", G * 4, &err); if (err) return cuda_fail(ctx, err, "scratch"); }
  }
  if (o->keep_values) {
    if (!p.o_perf) { p.o_perf = (double*)scratch(ctx, "perf", G * 8, &err); if (err) return cuda_fail(ctx, err, "scratch"); }
    if (!p.o_gain) { p.o_gain = (double*)scratch(ctx, "gain", G * 8, &err); if (err) return cuda_fail(ctx, err, "scratch"); }
  }
  if (o->kernel_rollup) {
    p.krec = (uint64_t*)scratch(ctx, "krec", std::max<uint64_t>(G, 1) * 8, &err);
    if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
  }
  const size_t plen = partials_len(*o);
  p.partials = (uint64_t*)scratch(ctx, "partials", plen * 8, &err);
  if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
  p.minmax = (uint64_t*)scratch(ctx, "minmax", 4 * 8, &err);
  if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
  init_partials<<<(unsigned)std::min<size_t>(64, (plen + 255) / 256), 256, 0, s>>>(p.partials, plen, p.minmax);
  ctx->launches++;
  // kernel attributes and occupancy are host calls on the launch path: set/queried once per
  // shared-memory size (the small tables of configs[2]/[3] are launch-latency bound)
  LSCAT_CUDA(ctx, ensure_smem_attr((const void*)reduce_groups_kernel, smem));
  LSCAT_CUDA(ctx, ensure_smem_attr((const void*)finalize_merged_kernel, smem_fin));
  const bool merge = ctx->world > 1 && o->point_sharded;
  const uint64_t warps_needed = (G + 31) / 32;
  const bool uniform = p.vec && p.rpg == 32;
  auto kern = uniform ? reduce_uniform32_kernel : reduce_groups_kernel;
  if (uniform) {
    smem = smem_hist + kUniStageBytes;
    LSCAT_CUDA(ctx, ensure_smem_attr((const void*)reduce_uniform32_kernel, smem));
  }
  int occ = 0;
  const auto ok = std::make_pair(uniform, smem);
  if (ctx->red_occ.empty()) {  // the selection chain's carve-out (stats.cu): no reconfiguration
    for (const void* f : {(const void*)reduce_groups_kernel, (const void*)reduce_uniform32_kernel,
                          (const void*)finalize_merged_kernel, (const void*)init_partials})
      LSCAT_CUDA(ctx, cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           (int)cudaSharedmemCarveoutMaxShared));
  }
  const auto it = ctx->red_occ.find(ok);
  if (it != ctx->red_occ.end()) {
    occ = it->second;
  } else {
    LSCAT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem));
    ctx->red_occ[ok] = occ;
  }
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctx->sm_count * std::max(occ, 1), (warps_needed + 7) / 8));
  p.acc_lo = 0;
  p.acc_hi = G;
  uint64_t own_lo = 0, own_hi = G;
  if (!merge) {
    p.mode = MODE_FUSED;
    if (G) kern<<<grid, 256, smem, s>>>(p), ctx->launches++;
    LSCAT_CUDA(ctx, cudaGetLastError());
  } else {
    // a9, point-sharded: per-group MIN(key) / MAX(l-code) / SUM(counts) over ranks, then each
    // rank accumulates its contiguous share of the groups.
    uint64_t* key = (uint64_t*)scratch(ctx, "g_key", G * 8, &err);
    if (err) return cuda_fail(ctx, err, "scratch");
    uint64_t* lc = (uint64_t*)scratch(ctx, "g_lcode", G * 8, &err);
    if (err) return cuda_fail(ctx, err, "scratch");
    uint32_t* cnt = (uint32_t*)scratch(ctx, "g_cnt", G * 12, &err);
    if (err) return cuda_fail(ctx, err, "scratch");
    p.g_key = key; p.g_lcode = lc; p.g_cnt = cnt;
    p.mode = MODE_GROUP_PARTIALS;
    if (G) kern<<<grid, 256, smem, s>>>(p), ctx->launches++;
    LSCAT_CUDA(ctx, cudaGetLastError());
    lscat_status ns = ctx->comm->allreduce(ctx, {{key, G, DT::U64, Op::Min}, {lc, G, DT::U64, Op::Max},
                                                 {cnt, 3 * G, DT::U32, Op::Sum}}, s);
    if (ns) return ns;
    own_lo = G * ctx->rank / ctx->world;
    own_hi = G * (ctx->rank + 1) / ctx->world;
    p.acc_lo = own_lo;
    p.acc_hi = own_hi;
    // reset accumulators written by the partial pass (none: partials untouched by mode 1
    // except zero-valued flushes), then finalize all groups, accumulating the owned range
    init_partials<<<(unsigned)std::min<size_t>(64, (plen + 255) / 256), 256, 0, s>>>(p.partials, plen, p.minmax);
    ctx->launches++;
    p.mode = MODE_FINALIZE_MERGED;
    const int g2 = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctx->sm_count * 4, (G + 255) / 256));
    if (G) finalize_merged_kernel<<<g2, 256, smem_fin, s>>>(p), ctx->launches++;
    LSCAT_CUDA(ctx, cudaGetLastError());
  }
  if (o->block_profile && G) {
    const size_t ML = (size_t)o->n_matrices * o->n_blocks;
    uint64_t* prof = p.partials + kNC + sh_words;  // [sum ML][count ML]
    const size_t psm = ML * 12;
    if (psm > 48 * 1024)
      LSCAT_CUDA(ctx, ensure_smem_attr((const void*)profile_kernel, psm));
    const int g3 = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctx->sm_count * 8, (G + 7) / 8));
    profile_kernel<<<g3, 256, psm, s>>>(p, p.o_bestrt, p.o_flags, prof, prof + ML);
    ctx->launches++;
    LSCAT_CUDA(ctx, cudaGetLastError());
  }
  if (o->kernel_rollup) {  // R-26, over the groups this rank accumulated
    RollupArgs q{};
    q.krec = p.krec;
    q.gkern = gkern;
    q.first_group = T->first_group;
    q.lo = p.acc_lo;
    q.hi = p.acc_hi;
    q.M = o->n_matrices;
    q.mshift = (q.M & (q.M - 1)) == 0 ? __builtin_ctz(q.M) : -1;
    q.nb = o->bins_per_unit;
    q.pln = o->perf_lt_num; q.pld = o->perf_lt_den; q.bln = o->band_lo_num; q.bld = o->band_lo_den;
    q.part = p.partials + plen - (8 + o->bins_per_unit + 1);
    const int W = ctx->world;
    uint64_t* bnd = (uint64_t*)scratch(ctx, "kbnd", (size_t)2 * kBndWords * 8 * (1 + W), &err);
    if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
    q.bnd = bnd;
    LSCAT_CUDA(ctx, cudaMemsetAsync(bnd, 0, 2 * kBndWords * 8, s));
    const size_t rsm = kRollupWords * 8 + (o->bins_per_unit + 1) * 4;
    if (rsm > 48 * 1024) LSCAT_CUDA(ctx, ensure_smem_attr((const void*)rollup_kernel, rsm));
    const uint64_t ng = q.hi - q.lo;
    // implicit ids, M a power of two <= 32: aligned-chunk kernel (LSCAT_ROLLUP_GENERAL=1: the
    // general segmented one, for A/B)
    static const bool general = getenv("LSCAT_ROLLUP_GENERAL") != nullptr;
    const bool uni = !q.gkern && q.mshift >= 0 && q.M <= 32 && !general;
    if (uni && rsm > 48 * 1024) LSCAT_CUDA(ctx, ensure_smem_attr((const void*)rollup_uniform_kernel, rsm));
    if (ng && uni) {
      const uint64_t nk = (ng + 2 * q.M) / q.M;  // kernels touched (upper bound)
      const int g4 = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctx->sm_count * 8, (nk + 255) / 256));
      rollup_uniform_kernel<<<g4, 256, rsm, s>>>(q);
      ctx->launches++;
      LSCAT_CUDA(ctx, cudaGetLastError());
    } else if (ng) {
      const int g4 = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctx->sm_count * 8, (ng + 255) / 256));
      rollup_kernel<<<g4, 256, rsm, s>>>(q);
      ctx->launches++;
      LSCAT_CUDA(ctx, cudaGetLastError());
    }
    uint64_t* all = bnd;
    if (W > 1) {
      all = bnd + 2 * kBndWords;
      lscat_status ns = ctx->comm->allgather(ctx, bnd, all, 2 * kBndWords, DT::U64, s);
      if (ns) return ns;
    }
    if (ctx->rank == 0) {
      rollup_boundary_kernel<<<1, 32, 0, s>>>(q, all, 2 * W);
      ctx->launches++;
      LSCAT_CUDA(ctx, cudaGetLastError());
    }
  }
  if (ctx->world > 1) {
    lscat_status ns = ctx->comm->allreduce(
        ctx, {{p.partials, plen, DT::U64, Op::Sum}, {p.minmax, 1, DT::U64, Op::Min},
              {p.minmax + 1, 1, DT::U64, Op::Max}, {p.minmax + 2, 1, DT::U64, Op::Min},
              {p.minmax + 3, 1, DT::U64, Op::Max}}, s);
    if (ns) return ns;
  }
  if (out->partials) LSCAT_CUDA(ctx, cudaMemcpyAsync(out->partials, p.partials, plen * 8, cudaMemcpyDeviceToDevice, s));
  // R-27: the percentile selection of opts->percentiles enqueued right behind the reduction
  // (one rank, not point-sharded, per-group values kept): lscat_stats with the same list only
  // collects it
  uint32_t early = EARLY_NONE;
  const double* perf_k = o->keep_values ? p.o_perf : out->perf;
  const double* gain_k = o->keep_values ? p.o_gain : out->gain;
  const uint64_t* partials_h = nullptr;
  if (o->n_percentiles && ctx->world == 1 && !o->point_sharded && G && perf_k && gain_k) {
    // lscat_stats follows: on small tables its host copy of the partials runs here, on a side
    // branch next to the one-launch selection instead of after it (configs[2]/[3])
    const bool side = G <= kEarlySmallGroups;
    if (side) {
      if (!ctx->aux_stream) {
        LSCAT_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
        LSCAT_CUDA(ctx, cudaEventCreateWithFlags(&ctx->aux_fork, cudaEventDisableTiming));
        LSCAT_CUDA(ctx, cudaEventCreateWithFlags(&ctx->aux_join, cudaEventDisableTiming));
      }
      uint64_t* hP = (uint64_t*)pinned(ctx, "stats_partials", plen * 8, &err);
      if (err) return cuda_fail(ctx, err, "reduce_table: pinned");
      LSCAT_CUDA(ctx, cudaEventRecord(ctx->aux_fork, s));
      LSCAT_CUDA(ctx, cudaStreamWaitEvent(ctx->aux_stream, ctx->aux_fork, 0));
      LSCAT_CUDA(ctx, cudaMemcpyAsync(hP, p.partials, plen * 8, cudaMemcpyDeviceToHost, ctx->aux_stream));
      LSCAT_CUDA(ctx, cudaEventRecord(ctx->aux_join, ctx->aux_stream));
      partials_h = hP;
    }
    lscat_status es = early_select(ctx, perf_k, gain_k, own_lo, own_hi, p.partials, p.minmax, o->bins_per_unit,
                                   o->percentiles, o->n_percentiles, s, &early);
    if (side) LSCAT_CUDA(ctx, cudaStreamWaitEvent(s, ctx->aux_join, 0));  // joined before any return
    if (es) return es;
    if (early != EARLY_SMALL) partials_h = nullptr;
  }
  ReduceState& rs = ctx->rs;
  rs.early = early;
  rs.partials_h = partials_h;
  rs.early_pct.assign(o->percentiles, o->percentiles + (early ? o->n_percentiles : 0));
  rs.valid = true;
  rs.opts = *o;
  rs.n_groups = G;
  rs.own_lo = own_lo;
  rs.own_hi = own_hi;
  rs.perf = o->keep_values ? p.o_perf : out->perf;
  rs.gain = o->keep_values ? p.o_gain : out->gain;
  rs.partials = p.partials;
  rs.minmax = p.minmax;
  if (T->mem == LSCAT_MEM_HOST) LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  return LSCAT_OK;
}

// Small device tables on one rank are launch-latency bound (configs[2]/[3]: ~5 dependent
// launches, memsets and copies for ~50 us of kernels): the sequence reduce_enqueue issues is
// captured once per argument set (the second call with the same arguments runs it normally
// and then captures the same calls into a graph) and later calls replay it with one
// cudaGraphLaunch.  A cached graph is used only while no scratch / pinned buffer has been
// (re)allocated since its capture.  LSCAT_REDUCE_NOGRAPH=1 disables it.
lscat_status lscat_reduce_table(lscat_ctx* ctx, const lscat_table* T, const lscat_reduce_opts* o,
                                lscat_reduce_out* out, void* stream) {
  using RedGraph = lscat_ctx::RedGraph;
  LSCAT_CHECK_CTX(ctx);
  static const bool no_graph = getenv("LSCAT_REDUCE_NOGRAPH") != nullptr;
  const bool graphable = !no_graph && ctx->world == 1 && T && opts_ok(o) && T->mem == LSCAT_MEM_DEVICE &&
                         T->n_groups > 0 && T->n_groups <= kEarlySmallGroups;
  if (!graphable) return reduce_enqueue(ctx, T, o, out, stream);
  std::string key;
  auto put = [&](const void* v, size_t n) { key.append(reinterpret_cast<const char*>(v), n); };
  put(T, sizeof *T);
  lscat_reduce_opts oc = *o;
  oc.percentiles = nullptr;  // by value below
  put(&oc, sizeof oc);
  if (o->n_percentiles) put(o->percentiles, o->n_percentiles * sizeof(double));
  lscat_reduce_out oo{};
  if (out) oo = *out;
  put(&oo, sizeof oo);
  put(&stream, sizeof stream);
  auto drop_oldest = [&]() {
    if (ctx->red_graphs.size() < 8) return;
    if (ctx->red_graphs.front().gx) cudaGraphExecDestroy(ctx->red_graphs.front().gx);
    ctx->red_graphs.erase(ctx->red_graphs.begin());
  };
  RedGraph* hit = nullptr;
  for (auto& rg : ctx->red_graphs)
    if (rg.key == key && rg.gen == ctx->scratch_gen) hit = &rg;
  if (hit && hit->gx) {
    LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));
    LSCAT_CUDA(ctx, cudaGraphLaunch(hit->gx, (cudaStream_t)stream));
    ctx->rs = hit->rs;
    ctx->rs.opts = *o;
    ctx->launches += hit->launches;
    return LSCAT_OK;
  }
  const uint64_t l0 = ctx->launches;
  lscat_status st = reduce_enqueue(ctx, T, o, out, stream);
  if (st || (hit && hit->tried)) return st;  // not capturable with these arguments
  const uint64_t gen = ctx->scratch_gen, l1 = ctx->launches;
  if (!hit) {  // first call with these arguments: remember them (per-call outputs never repeat)
    drop_oldest();
    RedGraph rg;
    rg.key = std::move(key);
    rg.gen = gen;
    ctx->red_graphs.push_back(std::move(rg));
    return LSCAT_OK;
  }
  // second call: capture the same sequence for the next ones
  const lscat::ReduceState rs = ctx->rs;
  hit->tried = true;
  cudaStream_t cs = ctx->capture_stream;
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    const lscat_status cst = reduce_enqueue(ctx, T, o, out, cs);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &g);
    cudaGraphExec_t gx = nullptr;
    if (!cst && ce == cudaSuccess && g && ctx->scratch_gen == gen && cudaGraphInstantiate(&gx, g, 0) == cudaSuccess) {
      hit->gx = gx;
      hit->rs = rs;
      hit->launches = l1 - l0;
    }
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();  // a capture that failed leaves no sticky error; the call itself succeeded
    if (cst && ctx->poisoned) return cst;
  }
  ctx->rs = rs;
  ctx->launches = l1;
  ctx->err.clear();
  return LSCAT_OK;
}

}  // extern "C"
