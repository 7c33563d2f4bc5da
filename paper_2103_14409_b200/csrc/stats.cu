// stats.cu — a10 (finalize the merged integer partials on the host) and a8 (exact
// nearest-rank percentiles of perf and gain over ratio-defined groups, R-13).
//
// Percentile selection is a multi-level radix select over the IEEE bit patterns of the
// positive doubles (bit order == value order), run entirely on the device:
//   sel_init    targets k = clamp(ceil(p * n_def)) from the merged partials, level-0 ranges
//               [min key, max key] per quantity (perf, gain);
//   sel_pass    one pass over the keys: for each open range (disjoint, sorted by lo; located by
//               binary search) either histogram the key into 8192 bins (bin 0 = {lo}, bin 1 =
//               (lo, base), bins 2.. uniform in key from base by a shift, last bin = {hi}) or,
//               when the range holds <= cap keys, gather it;
//   sel_resolve one CTA per range: scan its histogram (narrow each target to its bin) or sort
//               its gathered keys (bitonic, shared memory) and pick each target's rank;
//   (plan)      the last sel_resolve CTA merges the open targets into the next level's ranges.
// The host launches levels in batches of four and reads the state once per batch (one sync
// for the common case).  `base` skips the empty low binades of a level-0 range whose minimum
// is far below its maximum (gain = 0 next to gains of order 1).  With world > 1 the histograms
// are summed and the gathered keys all-gathered between sel_pass and sel_resolve, so every
// rank takes the same decisions.
#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "common.h"
#include "selbins.h"

namespace lscat {
namespace {

constexpr int kBins = 8192;           // bins per range and level
constexpr int kMaxT = 128;            // targets: 2 x <= 64 percentiles
constexpr int kMaxR = kMaxT;          // open ranges per level (<= open targets)
static_assert(kMaxR <= 128, "sel_pass range search covers 128 ranges");
constexpr int kSmemRanges = 2;        // histograms privatised in shared memory up to this many
constexpr int kLevelsPerBatch = 4;       // levels per host sync (large inputs)
constexpr int kLevelsPerBatchSmall = 2;  // up to kSmallKeys keys per quantity: level 0 narrows
constexpr uint64_t kSmallKeys = 1ull << 20;  // each target to a bin of a few hundred keys at most,
                                             // level 1 gathers and sorts it
constexpr uint64_t kGapKeys = 32ull << 52;  // 32 binades: keys below hi - kGapKeys share bin 1
constexpr uint64_t kNaNKey = 0x7FF8000000000000ull;
// Once the open ranges hold at most this many keys per quantity (and at most half of them), one
// pass copies them out and later levels read the copies instead of the full perf/gain arrays.
constexpr uint64_t kCompactCap = 1ull << 22;

struct Range {
  uint64_t lo, hi;   // inclusive key range
  uint64_t base;     // first key of the uniform bins
  uint64_t count;    // keys inside [lo, hi] over all ranks
  uint64_t span, g;  // hi - lo, base - lo (the pass works on d = k - lo)
  uint32_t shift, which, gather, pad;
};

struct Tgt {
  uint64_t lo, hi;   // current inclusive key range of the target
  uint64_t k;        // 1-based rank inside [lo, hi]
  uint64_t count;    // keys inside [lo, hi] over all ranks
  uint64_t key;      // result when done
  uint32_t which, done, range, pad;
};

struct SelState {
  uint32_t nt, nr, nw0, err;  // targets, open ranges, ranges of perf (sorted first), error code
  uint32_t open;              // targets still open after the last plan
  uint32_t src;               // 0: passes read perf/gain; 1: the compacted keys
  uint32_t compact;           // 1: the next pass also copies the keys it counts (src 0 only)
  uint32_t r0_valid;          // bit w: r0[w] holds quantity w's level-0 range
  uint32_t done_ctas;         // sel_resolve CTAs finished (the last one plans; reset to 0)
  uint32_t pad2;
  unsigned long long nc[2];   // compacted keys per quantity
  uint64_t n_def;
  uint32_t sampled_fail;      // the sampled first level missed a target (host falls back)
  uint32_t pad3;
  Range r0[2];                // level-0 ranges: later full passes filter keys by level-0 bin
  Range r[kMaxR];
  Tgt t[kMaxT];
};

struct PctArg {
  double p[kMaxT / 2];
};

// bin of a key inside the range, from d = k - lo (0 <= d <= span)
__device__ __forceinline__ int bin_of_d(const Range& R, uint64_t d) {
  if (d == 0) return 0;
  if (d == R.span) return kBins - 1;
  if (d < R.g) return 1;
  return 2 + (int)((d - R.g) >> R.shift);
}

// inclusive key range of bin b of range R (the inverse of bin_of_d)
__device__ __forceinline__ void bin_keys(const Range& R, int b, uint64_t* lo, uint64_t* hi) {
  if (b == 0) {
    *lo = *hi = R.lo;
  } else if (b == kBins - 1) {
    *lo = *hi = R.hi;
  } else if (b == 1) {
    *lo = R.lo + 1;
    *hi = R.base - 1;
  } else {
    *lo = R.base + ((uint64_t)(b - 2) << R.shift);
    const uint64_t top = R.base + ((uint64_t)(b - 1) << R.shift) - 1;  // may wrap only past hi
    *hi = (top < *lo || top > R.hi - 1) ? R.hi - 1 : top;
  }
}

__device__ Range make_range(uint64_t lo, uint64_t hi, uint64_t count, uint32_t which, uint32_t cap) {
  Range R;
  R.lo = lo;
  R.hi = hi;
  R.count = count;
  R.which = which;
  R.gather = count <= cap;
  R.pad = 0;
  R.base = (hi > kGapKeys && hi - kGapKeys > lo + 1) ? hi - kGapKeys : lo + 1;
  uint32_t s = 0;
  if (R.base < hi) {
    // the smallest s with (span >> s) <= kBins - 4, span = the largest (k - base) of a middle
    // key: from the bit lengths, then at most one step (every thread of sel_small runs this,
    // a shift-by-one loop cost up to ~50 dependent iterations per quantity)
    const uint64_t span = hi - 1 - R.base;
    constexpr uint64_t M = (uint64_t)(kBins - 4);
    if (span > M) {
      s = (uint32_t)((64 - __clzll((long long)span)) - (64 - __clzll((long long)M)));
      if ((span >> s) > M) s++;
    }
  }
  R.shift = s;
  R.span = hi - lo;
  R.g = R.base - lo;
  return R;
}

__device__ __forceinline__ uint64_t t_count(const SelState* st, int i) { return st->t[i].count; }

// Merge the open targets into disjoint ranges sorted by (which, lo).  One CTA; thread i < nt
// owns target i.  Called by sel_init and by the last CTA of sel_resolve.
__device__ void plan_ranges_warp(SelState* st, uint32_t cap, int nt);

__device__ void plan_ranges(SelState* st, uint32_t cap) {
  __shared__ uint64_t slo[kMaxT], shi[kMaxT];
  __shared__ uint32_t sw[kMaxT], sopen[kMaxT], sfirst[kMaxT];
  const int i = threadIdx.x;
  const int nt = (int)st->nt;
  if (nt <= 32) {  // one warp (every thread of the CTA calls this)
    if (i < 32) plan_ranges_warp(st, cap, nt);
    __syncthreads();
    return;
  }
  bool open = false;
  if (i < nt) {
    Tgt& t = st->t[i];
    if (!t.done && t.lo == t.hi) { t.done = 1; t.key = t.lo; }
    open = !t.done;
    slo[i] = t.lo;
    shi[i] = t.hi;
    sw[i] = t.which;
  }
  if (i < kMaxT) sopen[i] = open;
  __syncthreads();
  bool first = open;
  if (open)
    for (int j = 0; j < i; j++)
      if (sopen[j] && sw[j] == sw[i] && slo[j] == slo[i] && shi[j] == shi[i]) { first = false; break; }
  if (i < kMaxT) sfirst[i] = first;
  __syncthreads();
  uint32_t rank = 0, nr = 0, nw0 = 0, nopen = 0;
  for (int j = 0; j < nt; j++) {
    nopen += sopen[j];
    if (!sfirst[j]) continue;
    nr++;
    nw0 += sw[j] == 0;
    if (open && (sw[j] < sw[i] || (sw[j] == sw[i] && slo[j] < slo[i]))) rank++;
  }
  if (open) {
    Tgt& t = st->t[i];
    t.range = rank;
    if (first) st->r[rank] = make_range(t.lo, t.hi, t.count, t.which, cap);
  }
  __shared__ unsigned long long s_keys[2];
  if (i < 2) s_keys[i] = 0;
  __syncthreads();
  if (open && first && !st->r[rank].gather) atomicAdd(&s_keys[st->r[rank].which], (unsigned long long)t_count(st, i));
  __syncthreads();
  if (i == 0) {
    st->nr = nr;
    st->nw0 = nw0;
    st->open = nopen;
    if (st->compact) {  // the pass that just ran copied the keys: read the copies from now on
      st->src = 1;
      st->compact = 0;
    } else if (st->src == 0 && nr > 0 && s_keys[0] <= kCompactCap && s_keys[1] <= kCompactCap &&
               2 * (s_keys[0] + s_keys[1]) <= st->n_def) {
      st->compact = 1;
      st->nc[0] = st->nc[1] = 0;
    }
  }
}

// plan_ranges for <= 32 targets in one warp (lane i = target i): the same ranges, range ids
// (rank by (which, lo) among the first occurrences) and counters, from match_any / ballot and
// shuffles instead of O(nt^2) shared-memory loops between barriers.
__device__ void plan_ranges_warp(SelState* st, uint32_t cap, int nt) {
  const unsigned FULL = 0xffffffffu;
  const int i = threadIdx.x;
  const bool act = i < nt;
  uint64_t lo = 0, hi = 0, cnt = 0;
  uint32_t w = 0;
  bool open = false;
  if (act) {
    Tgt& t = st->t[i];
    if (!t.done && t.lo == t.hi) { t.done = 1; t.key = t.lo; }
    open = !t.done;
    lo = t.lo;
    hi = t.hi;
    w = t.which;
    cnt = t.count;
  }
  const unsigned m = __match_any_sync(FULL, lo) & __match_any_sync(FULL, hi) &
                     __match_any_sync(FULL, open ? w : 2u + (uint32_t)i);
  const bool first = open && __ffs(m) - 1 == i;
  const unsigned firsts = __ballot_sync(FULL, first);
  const uint32_t nr = (uint32_t)__popc(firsts);
  const uint32_t nw0 = (uint32_t)__popc(__ballot_sync(FULL, first && w == 0));
  const uint32_t nopen = (uint32_t)__popc(__ballot_sync(FULL, open));
  uint32_t rank = 0;
  for (unsigned f = firsts; f; f &= f - 1) {  // warp-uniform
    const int j = __ffs(f) - 1;
    const uint32_t wj = __shfl_sync(FULL, w, j);
    const uint64_t lj = __shfl_sync(FULL, lo, j);
    rank += (wj < w || (wj == w && lj < lo)) ? 1u : 0u;
  }
  bool gather = true;
  if (open) {
    st->t[i].range = rank;
    if (first) {
      const Range R = make_range(lo, hi, cnt, w, cap);
      st->r[rank] = R;
      gather = R.gather;
    }
  }
  // keys of the non-gather ranges per quantity (the compaction decision below)
  unsigned long long k0 = (first && !gather && w == 0) ? cnt : 0ull, k1 = (first && !gather && w == 1) ? cnt : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    k0 += __shfl_xor_sync(FULL, k0, o);
    k1 += __shfl_xor_sync(FULL, k1, o);
  }
  if (i == 0) {
    st->nr = nr;
    st->nw0 = nw0;
    st->open = nopen;
    if (st->compact) {  // the pass that just ran copied the keys: read the copies from now on
      st->src = 1;
      st->compact = 0;
    } else if (st->src == 0 && nr > 0 && k0 <= kCompactCap && k1 <= kCompactCap && 2 * (k0 + k1) <= st->n_def) {
      st->compact = 1;
      st->nc[0] = st->nc[1] = 0;
    }
  }
}

__global__ void __launch_bounds__(kMaxT) sel_init(SelState* st, const uint64_t* __restrict__ partials,
                                                  const uint64_t* __restrict__ mm, PctArg pct, uint32_t npct,
                                                  uint32_t cap) {
  const int i = threadIdx.x;
  const uint64_t n_def = partials[LSCAT_P_RATIO_DEFINED];
  if (i == 0) {
    st->nt = 2 * npct;
    st->err = 0;
    st->done_ctas = 0;
    st->src = 0;
    st->compact = 0;
    st->n_def = n_def;
  }
  if (i < (int)(2 * npct)) {
    Tgt t{};
    t.which = i >= (int)npct;
    const double r = ceil(pct.p[i % npct] * (double)n_def);  // nearest rank (R-13)
    t.k = r < 1.0 ? 1 : (r > (double)n_def ? n_def : (uint64_t)r);
    t.lo = mm[2 * t.which];
    t.hi = mm[2 * t.which + 1];
    t.count = n_def;
    t.done = n_def == 0;
    t.key = kNaNKey;
    st->t[i] = t;
  }
  __syncthreads();
  plan_ranges(st, cap);
  __syncthreads();
  if (i == 0) {  // remember the level-0 range of each quantity (the bin filter of later passes)
    uint32_t v = 0;
    for (uint32_t j = 0; j < st->nr; j++) {
      const uint32_t w = st->r[j].which;
      if (!st->r[j].gather && !(v & (1u << w))) { st->r0[w] = st->r[j]; v |= 1u << w; }
    }
    st->r0_valid = v;
  }
}


// One pass over this rank's values (src 0: perf/gain[lo, hi); src 1: the compacted keys).
// cand = [kMaxR counts][kMaxR x cap keys]; cbuf = [2][kCompactCap] compacted keys.
// kSmem (level 0 only: one range per quantity): histograms privatised in shared memory, the two
// single-key end bins (perf == 1.0, gain == 0, the extremes) counted with one ballot per warp.
// Otherwise (levels >= 1: narrow ranges, few hits) global atomics aggregated per warp over
// equal bins (match.any), so a heavily repeated value does not serialise on one address.
// Keys are the raw bit patterns: NaN (undefined group) patterns exceed every finite range.
// largest power of two < n (0 for n <= 1): the first step of the range search
__device__ __forceinline__ uint32_t top_step(uint32_t n) { return n > 1 ? 1u << (31 - __clz(n - 1)) : 0u; }

// Levels >= 1, a warp with at least one key inside an open range: gather, histogram
// (match.any-aggregated global atomics), or -- on the copy-only level that starts compaction --
// a warp-aggregated copy of the keys.  Out of line so the unrolled scan loop
// of sel_pass stays small enough for the instruction cache.  Called by all 32 lanes.
constexpr uint32_t kStageKeys = 1024;  // per quantity and CTA: compaction staged in smem

__device__ __noinline__ void hit_slow(const Range* sr, uint32_t r, uint64_t k, uint64_t d, bool hit, int w,
                                      int lane, uint32_t* __restrict__ hist,
                                      unsigned long long* __restrict__ cand, uint32_t cap, bool compact,
                                      SelState* __restrict__ st, double* __restrict__ cbuf,
                                      uint64_t* __restrict__ stage, uint32_t* __restrict__ s_nc) {
  const unsigned FULL = 0xffffffffu;
  const Range& R = sr[r];
  // lanes may sit in different ranges (gathered or histogrammed): no early exit before the
  // warp collectives below
  {  // gather (<= cap keys in the whole range): one counter atomic per range and warp
    const bool g = hit && R.gather;
    const unsigned peers = __match_any_sync(FULL, g ? r : 0xFFFFFFFFu);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (g && lane == leader) base = atomicAdd(&cand[r], (unsigned long long)__popc(peers));
    base = __shfl_sync(FULL, base, leader);
    if (g) {
      const unsigned long long idx = base + __popc(peers & ((1u << lane) - 1u));
      if (idx < cap) cand[kMaxR + (size_t)r * cap + idx] = k;
    }
  }
  const bool counted = hit && !R.gather;
  if (!compact) {
    const int key = counted ? (int)(r * kBins) + bin_of_d(R, d) : -1;
    const unsigned peers = __match_any_sync(FULL, key);
    if (counted && (__ffs(peers) - 1) == lane) atomicAdd(&hist[key], (uint32_t)__popc(peers));
  } else {  // copy-only level: the keys of the open ranges are copied out, not histogrammed
            // (the next level histograms the copies with the same ranges)
    // staged in the CTA's shared buffer (one shared atomic per warp); the CTA reserves its
    // global range once at the end (sel_pass), so the global counter is not a hot spot
    const unsigned m = __ballot_sync(FULL, counted);
    uint32_t at = 0;
    if (m && lane == 0) at = atomicAdd(&s_nc[w], (uint32_t)__popc(m));
    at = __shfl_sync(FULL, at, 0);
    const uint32_t pos = at + __popc(m & ((1u << lane) - 1u));
    if (counted) {
      if (pos < kStageKeys) {
        stage[(size_t)w * kStageKeys + pos] = k;
      } else {  // stage full: straight to the global buffer
        const unsigned long long g = atomicAdd(&st->nc[w], 1ull);
        if (g < kCompactCap) reinterpret_cast<uint64_t*>(cbuf)[(size_t)w * kCompactCap + g] = k;
      }
    }
  }
}

template <bool kSmem, int kT, int kU = 8>
__global__ void __launch_bounds__(kT, kSmem ? 2 : 4) sel_pass(const double* __restrict__ perf, const double* __restrict__ gain,
                                               uint64_t lo, uint64_t hi, SelState* __restrict__ st,
                                               uint32_t* __restrict__ hist, unsigned long long* __restrict__ cand,
                                               uint32_t cap, double* __restrict__ cbuf) {
  __shared__ Range sr[kMaxR];
  extern __shared__ uint32_t sh_hist[];
  const uint32_t nr = st->nr;
  if (nr == 0) return;
  const uint32_t nw0 = st->nw0, nw1 = nr - nw0;
  if (kSmem && (nw0 > 1 || nw1 > 1)) {  // host contract: level 0 only
    if (threadIdx.x == 0) atomicOr(&st->err, 8u);
    return;
  }
  const bool compact = !kSmem && st->compact;
  uint64_t hi0 = hi, hi1 = hi;
  if (!kSmem && st->src) {
    perf = cbuf;
    gain = cbuf + kCompactCap;
    lo = 0;
    hi0 = st->nc[0];
    hi1 = st->nc[1];
  }
  for (uint32_t i = threadIdx.x; i < nr; i += kT) sr[i] = st->r[i];
  if (kSmem)
    for (uint32_t i = threadIdx.x; i < nr * kBins; i += kT) sh_hist[i] = 0;
  // Levels >= 1 over the full arrays: a coarse bitmap per quantity over the high key bits,
  // cell = (k >> S) - (lo0 >> S) with S >= 32 chosen so the level-0 range [lo0, hi0] spans at
  // most kCells cells; a cell is marked if any open range touches it.  A key whose cell is
  // unmarked is in no open range, so the range search (and its vote) is skipped for it with a
  // handful of 32-bit instructions on the key's high word.
  constexpr uint32_t kCells = 1u << 16;
  __shared__ uint32_t bm[2][kCells / 32];
  __shared__ uint32_t s_filt;
  __shared__ uint64_t stage[kSmem ? 1 : 2 * kStageKeys];
  __shared__ uint32_t s_nc[2];
  __shared__ unsigned long long s_base[2];
  if (threadIdx.x < 2) s_nc[threadIdx.x] = 0;
  uint32_t filt = (!kSmem && !st->src) ? st->r0_valid : 0u;
  uint32_t fsh[2] = {0, 0}, fbase[2] = {0, 0};  // S - 32 and (lo0 >> S) per quantity
  if (filt) {
#pragma unroll
    for (int w = 0; w < 2; w++) {
      if (!(filt & (1u << w))) continue;
      const uint64_t lo0 = st->r0[w].lo, hi0 = st->r0[w].hi;
      uint32_t S = 32;
      while (((hi0 >> S) - (lo0 >> S)) >= kCells) S++;
      fsh[w] = S - 32;
      fbase[w] = (uint32_t)(lo0 >> S);
    }
    for (uint32_t i = threadIdx.x; i < 2 * (kCells / 32); i += kT) (&bm[0][0])[i] = 0u;
  }
  if (threadIdx.x == 0) s_filt = filt;
  __syncthreads();
  if (filt)
    for (uint32_t i = threadIdx.x; i < nr; i += kT) {
      const Range& R = sr[i];
      const uint32_t w = R.which;
      if (!(filt & (1u << w))) continue;
      const uint32_t S = (w ? fsh[1] : fsh[0]) + 32, b0 = w ? fbase[1] : fbase[0];
      const uint64_t c_lo = (R.lo >> S) - b0, c_hi = (R.hi >> S) - b0;
      if (c_lo > c_hi || c_hi >= kCells) {  // outside the level-0 range: no filter for w
        atomicAnd(&s_filt, ~(1u << w));
        continue;
      }
      for (uint32_t cc = (uint32_t)c_lo; cc <= (uint32_t)c_hi; cc++) atomicOr(&bm[w][cc >> 5], 1u << (cc & 31));
    }
  __syncthreads();
  filt = s_filt;
  const uint32_t* bmp[2] = {bm[0], bm[1]};
  uint32_t c0[2] = {0, 0}, cL[2] = {0, 0};  // level 0: end-bin counts per thread
  Range sr0[2];  // level 0: the range of each quantity, kept in registers
  if (kSmem) {
    sr0[0] = sr[0];
    sr0[1] = sr[nw0 ? nw0 : 0];
  }
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint64_t end = hi0 > hi1 ? hi0 : hi1;
  // A warp takes kU chunks of 32 consecutive keys per iteration and issues all loads before
  // using them; arrays with no open range are not read.  (kU = 1 for small inputs: more warps,
  // each with a shorter latency-bound critical path.)
  const uint64_t wstride = (uint64_t)gridDim.x * kT * kU;
  for (uint64_t base = lo + (blockIdx.x * (uint64_t)kT + (threadIdx.x & ~31u)) * kU; base < end;
       base += wstride) {
    uint64_t v[2][kU];
#pragma unroll
    for (int w = 0; w < 2; w++) {
      const uint64_t* src = reinterpret_cast<const uint64_t*>(w ? gain : perf) + base + lane;
      const uint64_t hw = (w ? hi1 : hi0) - base;  // keys left in this array (if > 0)
      const bool rd = (w ? nw1 : nw0) && (w ? hi1 : hi0) > base;
      const bool full = rd && hw >= 32 * kU;
#pragma unroll
      for (int u = 0; u < kU; u++)
        v[w][u] = (full || (rd && (uint64_t)(32 * u + lane) < hw)) ? __ldg(src + 32 * u) : kNaNKey;
    }
    if (kSmem) {
#pragma unroll
      for (int u = 0; u < kU; u++) {
#pragma unroll
        for (int w = 0; w < 2; w++) {
          const uint32_t nw = w ? nw1 : nw0;
          if (!nw) continue;  // uniform
          const uint64_t k = v[w][u];
          const uint32_t b0 = w ? nw0 : 0;
          // level 0: one range per quantity (registers); end bins counted per thread
          const Range& R = sr0[w];
          const uint64_t d = k - R.lo;
          const bool hit = d <= R.span;  // k < lo wraps d past every span (< 2^63)
          if (R.gather) {                // uniform: one counter atomic per warp
            const unsigned m = __ballot_sync(FULL, hit);
            if (m) {
              const int leader = __ffs(m) - 1;
              unsigned long long base = 0;
              if (lane == leader) base = atomicAdd(&cand[b0], (unsigned long long)__popc(m));
              base = __shfl_sync(FULL, base, leader);
              if (hit) {
                const unsigned long long idx = base + __popc(m & ((1u << lane) - 1u));
                if (idx < cap) cand[kMaxR + (size_t)b0 * cap + idx] = k;
              }
            }
            continue;
          }
          int b = 2 + (int)((d - R.g) >> R.shift);
          b = d < R.g ? 1 : b;
          const bool is0 = hit && d == 0, isL = hit && d == R.span;
          c0[w] += is0;
          cL[w] += isL;
          if (hit && !is0 && !isL) atomicAdd(&sh_hist[b0 * kBins + b], 1u);
        }
      }
      continue;
    }
    // levels >= 1: first a branch-free candidate mask over the 2 x kU keys of each lane (the
    // coarse cell bitmap, or every key when unfiltered), one vote for the whole batch; the
    // range search and its per-key vote run only for key slots some lane flagged
    uint32_t m = 0;
#pragma unroll
    for (int u = 0; u < kU; u++)
#pragma unroll
      for (int w = 0; w < 2; w++) {
        const uint32_t nw = w ? nw1 : nw0;
        uint32_t c = nw != 0;
        if (filt & (1u << w)) {  // branch-free: clamp the cell, mask the out-of-range case
          const uint32_t cell = ((uint32_t)(v[w][u] >> 32) >> fsh[w]) - fbase[w];
          const uint32_t cl = min(cell, kCells - 1);
          c = (bmp[w][cl >> 5] >> (cl & 31)) & (uint32_t)(cell < kCells);
        }
        m |= c << (2 * u + w);
      }
    const uint32_t mall = __reduce_or_sync(FULL, m);  // warp-uniform: slots some lane flagged
    if (!mall) continue;
#pragma unroll
    for (int u = 0; u < kU; u++) {
#pragma unroll
      for (int w = 0; w < 2; w++) {
        if (!((mall >> (2 * u + w)) & 1u)) continue;
        const uint32_t nw = w ? nw1 : nw0;
        const uint64_t k = v[w][u];
        const uint32_t b0 = w ? nw0 : 0;
        // last range with lo <= k (ranges sorted by lo): binary lifting with a warp-uniform
        // trip count, not unrolled (keeps the 16 unrolled copies small)
        uint32_t r = b0;
#pragma unroll 1
        for (uint32_t h = top_step(nw); h; h >>= 1) {
          const uint32_t q = r + h;
          const bool ok = q < b0 + nw;
          const uint64_t ql = sr[ok ? q : r].lo;
          r = (ok && ql <= k) ? q : r;
        }
        const Range& R = sr[r];
        const uint64_t d = k - R.lo;
        const bool hit = d <= R.span;  // k < lo wraps d past every span (< 2^63)
        if (!__any_sync(FULL, hit)) continue;
        hit_slow(sr, r, k, d, hit, w, lane, hist, cand, cap, compact, st, cbuf, stage, s_nc);
      }
    }
  }
  if (!kSmem && compact) {  // flush the staged compaction: one global reservation per quantity
    __syncthreads();
    if (threadIdx.x < 2) {
      const uint32_t n = min(s_nc[threadIdx.x], kStageKeys);
      s_base[threadIdx.x] = n ? atomicAdd(&st->nc[threadIdx.x], (unsigned long long)n) : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < 2; w++) {
      const uint32_t n = min(s_nc[w], kStageKeys);
      for (uint32_t i = threadIdx.x; i < n; i += kT) {
        const unsigned long long g = s_base[w] + i;
        if (g < kCompactCap) reinterpret_cast<uint64_t*>(cbuf)[(size_t)w * kCompactCap + g] = stage[w * kStageKeys + i];
      }
    }
  }
  if (kSmem) {
#pragma unroll
    for (int w = 0; w < 2; w++) {
      const uint32_t a = __reduce_add_sync(FULL, c0[w]), z = __reduce_add_sync(FULL, cL[w]);
      const uint32_t b0 = w ? nw0 : 0;
      if (lane == 0 && (w ? nw1 : nw0)) {
        if (a) atomicAdd(&sh_hist[b0 * kBins], a);
        if (z) atomicAdd(&sh_hist[b0 * kBins + kBins - 1], z);
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nr * kBins; i += kT)
      if (sh_hist[i]) atomicAdd(&hist[i], sh_hist[i]);
  }
}

// One CTA per open range.  Histogram ranges: narrow every target of the range to the bin that
// holds its rank, then zero the histogram for the next level.  Gathered ranges: sort the keys
// of all ranks and pick.  cand_all = world x [kMaxR counts][kMaxR x cap keys].
__device__ void resolve_range(SelState* st, uint32_t* __restrict__ hist,
                              const unsigned long long* __restrict__ cand_all,
                              unsigned long long* __restrict__ cand_own, int world, uint32_t cap) {
  extern __shared__ unsigned long long sk[];
  __shared__ unsigned long long wsum[32];
  __shared__ unsigned long long s_total;
  __shared__ unsigned long long s_k[kMaxT];
  const uint32_t r = blockIdx.x;
  const Range R = st->r[r];
  const int nt = (int)st->nt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!R.gather) {
    if (st->compact) return;  // copy-only level: nothing was counted, the ranges stand
    constexpr int kPer = kBins / 1024;
    uint32_t* h = hist + (size_t)r * kBins;
    uint32_t c[kPer];
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < kPer; j++) { c[j] = h[tid * kPer + j]; sum += c[j]; }
#pragma unroll
    for (int j = 0; j < kPer; j++) h[tid * kPer + j] = 0;
    unsigned long long inc = sum;  // block-wide inclusive scan of the per-thread sums
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      unsigned long long x = wsum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      wsum[lane] = x;
      if (lane == 31) s_total = x;
    }
    __syncthreads();
    const unsigned long long ex = inc - sum + (warp ? wsum[warp - 1] : 0ull);
    if (tid == 0 && s_total != R.count) atomicOr(&st->err, 1u);  // keys lost or double-counted
    // snapshot the ranks before any thread rewrites a target
    if (tid < nt) {
      const Tgt& t = st->t[tid];
      s_k[tid] = (t.done || t.range != r) ? 0ull : t.k;
    }
    __syncthreads();
    for (int i = 0; i < nt; i++) {
      const uint64_t k = s_k[i];
      if (!(k && ex < k && k <= ex + sum)) continue;
      Tgt& t = st->t[i];
      unsigned long long cum = ex;
      int j = 0;
      while (cum + c[j] < k) cum += c[j++];
      const int b = tid * kPer + j;
      t.k = k - cum;
      t.count = c[j];
      bin_keys(R, b, &t.lo, &t.hi);
    }
  } else {
    const size_t stride = (size_t)kMaxR * (cap + 1);
    unsigned long long total = 0;
    for (int w = 0; w < world; w++) total += min(cand_all[(size_t)w * stride + r], (unsigned long long)cap);
    if (total != R.count || total > cap) {
      if (tid == 0) atomicOr(&st->err, 2u);
      return;
    }
    uint32_t P = 1;
    while (P < total) P <<= 1;
    uint32_t at = 0;
    for (int w = 0; w < world; w++) {
      const unsigned long long* seg = cand_all + (size_t)w * stride;
      const uint32_t c = (uint32_t)min(seg[r], (unsigned long long)cap);
      for (uint32_t i = tid; i < c; i += blockDim.x) sk[at + i] = seg[kMaxR + (size_t)r * cap + i];
      at += c;
    }
    for (uint32_t i = at + tid; i < P; i += blockDim.x) sk[i] = ~0ull;
    __syncthreads();
    for (uint32_t kk = 2; kk <= P; kk <<= 1)
      for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < P; i += blockDim.x) {
          const uint32_t ixj = i ^ j;
          if (ixj > i) {
            const unsigned long long a = sk[i], b = sk[ixj];
            if ((a > b) == ((i & kk) == 0)) { sk[i] = b; sk[ixj] = a; }
          }
        }
        __syncthreads();
      }
    if (tid == 0) {
      for (int i = 0; i < nt; i++) {
        Tgt& t = st->t[i];
        if (t.done || t.range != r) continue;
        if (t.k == 0 || t.k > total) { atomicOr(&st->err, 4u); continue; }
        t.key = sk[t.k - 1];
        t.lo = t.hi = t.key;
        t.done = 1;
      }
      cand_own[r] = 0;
    }
  }
}

// sel_resolve: one CTA per open range (resolve_range); the last CTA to finish then plans the
// next level's ranges (plan_ranges), so a level is two launches (pass, resolve) instead of three.
// Every early exit inside resolve_range is CTA-uniform.
__global__ void __launch_bounds__(1024) sel_resolve(SelState* st, uint32_t* __restrict__ hist,
                                                    const unsigned long long* __restrict__ cand_all,
                                                    unsigned long long* __restrict__ cand_own, int world,
                                                    uint32_t cap) {
  __shared__ bool s_last;
  if (blockIdx.x < st->nr) resolve_range(st, hist, cand_all, cand_own, world, cap);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&st->done_ctas, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) st->done_ctas = 0;
  if (st->nr) plan_ranges(st, cap);
}

// ---- sampled first level (large inputs) -----------------------------------------------
// Instead of a histogram pass followed by a compaction pass over perf/gain, one pass counts
// every key exactly against sample-planned intervals of the fixed bins of selbins.h and copies
// the keys inside them (R-27):
//   sample  runs of kSampleRun consecutive keys at kSampleRuns evenly spaced positions (~2^20
//           keys, 128-byte reads), histogrammed over the fixed bins;
//   plan    every target's window of sample ranks (rank ~ p ns, +- 4.5 sqrt(.) + 32) as bins,
//           merged per quantity into <= kIvQ sorted disjoint intervals; the bins inside get an
//           exact-count slot each, the bins between intervals share one gap counter;
//   pass    every counted key (perf < 1, finite gain > 0; the single-valued bins perf == 1 <=>
//           gain == 0 are the reducer's perf_hist[nb]) adds 1 to its slot or gap and the slot
//           keys are copied;
//   check   the exact counts in key order (gap 0, interval 0's bins, gap 1, ...) locate every
//           target: inside a slot it is narrowed to that fixed bin, whose keys all sit in the
//           copies; in a gap (a sampling miss) or with overflowing copies the selection
//           restarts on the histogram path, so the result never depends on the sample.
constexpr int kIvQ = 9;                        // intervals per quantity (<= percentiles)
constexpr uint32_t kSpSlots = 1024;            // exact-count bins per quantity
constexpr uint32_t kSpCnt = kSpSlots + kIvQ + 1;  // slots, then gaps 0..niv
constexpr uint32_t kSpSlotFlag = 0x8000u;      // map entry: slot (else: the gap index)
constexpr uint64_t kSampleRuns = 1 << 16;      // sampled positions ...
constexpr uint32_t kSampleRun = 16;            // ... of 16 consecutive keys each
constexpr uint32_t kSpStage = 96;              // per warp and quantity: copies staged in smem
static_assert(kIvQ + 1 <= 10, "ten gap fields in two redux words");

struct SampPlan {
  uint32_t fail, pad;
  uint32_t niv[2], nslot[2];                   // intervals, slots used per quantity
  uint32_t b1[2][kIvQ], b2[2][kIvQ];           // fixed-bin intervals (inclusive), sorted, disjoint
  uint32_t slot0[2][kIvQ];                     // slot of each interval's first bin
  unsigned long long ncopy[2];                 // keys copied (this rank)
  unsigned long long ncopy_all[2];             // keys copied over all ranks (overflow check)
  uint32_t cnt[2][kSpCnt];                     // exact counts: slots, then gaps
  uint16_t map[2][kFxBins];                    // per fixed bin: kSpSlotFlag | slot, or its gap
  unsigned long long stamp[6];                 // %globaltimer in sel_plan_sampled (debug)
};

// Programmatic dependent launch between the sampled path's kernels on one rank: the next kernel
// is launched while its producer drains and waits here for the producer's completion and
// memory (no early trigger: the kernels never overlap).  A no-op without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ bool valid_key(uint64_t k) { return k < 0x7FF0000000000000ull; }
__device__ __forceinline__ bool virtual_bin(uint32_t w, uint32_t b) { return w == 0 ? b == kFxBins - 2 : b == 0; }
__device__ __forceinline__ uint32_t fx_bin(uint32_t w, uint64_t k) { return w == 0 ? fx_perf_bin(k) : fx_gain_bin(k); }

// Sample histogram over the fixed bins (the single-valued bins included).  Thread j reads key
// (j % kSampleRun) of run j / kSampleRun.
__global__ void __launch_bounds__(256) sel_sample_hist(const double* __restrict__ perf,
                                                       const double* __restrict__ gain, uint64_t lo,
                                                       uint64_t hi, uint64_t rstride,
                                                       uint32_t* __restrict__ shist) {
  __shared__ uint32_t h[2 * kFxBins];
  for (uint32_t i = threadIdx.x; i < 2 * kFxBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  // four samples of each quantity in flight per thread (the loop is load-latency bound)
  constexpr int kV = 4;
  const uint64_t total = kSampleRuns * kSampleRun, T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j0 < total; j0 += kV * T) {
    uint64_t kp[kV], kg[kV];
#pragma unroll
    for (int v = 0; v < kV; v++) {
      const uint64_t j = j0 + v * T;
      const uint64_t i = lo + (j / kSampleRun) * rstride + (j % kSampleRun);
      const bool in = j < total && i < hi;
      kp[v] = in ? (uint64_t)__double_as_longlong(__ldcs(perf + i)) : kNaNKey;
      kg[v] = in ? (uint64_t)__double_as_longlong(__ldcs(gain + i)) : kNaNKey;
    }
#pragma unroll
    for (int v = 0; v < kV; v++) {
      if (valid_key(kp[v])) atomicAdd(&h[fx_perf_bin(kp[v])], 1u);
      if (valid_key(kg[v])) atomicAdd(&h[kFxBins + fx_gain_bin(kg[v])], 1u);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 2 * kFxBins; i += blockDim.x)
    if (h[i]) atomicAdd(&shist[i], h[i]);
}

// Inclusive scan of a quantity's kFxBins counts into pre[] (1024 threads; part: 32 + 1024 words
// of scratch).
__device__ void scan_bins(const uint32_t* __restrict__ c_in, unsigned long long virt, uint32_t w,
                          unsigned long long* pre, unsigned long long* part) {
  constexpr int kPer = (kFxBins + 1023) / 1024;
  const int tid = threadIdx.x;
  unsigned long long c[kPer], sum = 0;
#pragma unroll
  for (int j = 0; j < kPer; j++) {
    const uint32_t b = (uint32_t)tid * kPer + j;
    c[j] = b < kFxBins ? (virtual_bin(w, b) ? virt : (unsigned long long)c_in[b]) : 0ull;
    sum += c[j];
  }
  // warp-shuffle scan of the per-thread sums, then of the 32 warp totals (part[0..31])
  const int lane = tid & 31, wid = tid >> 5;
  unsigned long long inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) part[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    unsigned long long x = part[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    part[lane] = x;
  }
  __syncthreads();
  part[32 + tid] = inc + (wid ? part[wid - 1] : 0ull);  // inclusive scan of the thread sums
  unsigned long long run = part[32 + tid] - sum;
#pragma unroll
  for (int j = 0; j < kPer; j++) {
    const uint32_t b = (uint32_t)tid * kPer + j;
    run += c[j];
    if (b < kFxBins) pre[b] = run;
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t first_reaching(const unsigned long long* P, unsigned long long x) {
  uint32_t a = 0, b = kFxBins - 1;  // smallest b with P[b] >= x
  while (a < b) {
    const uint32_t m = (a + b) / 2;
    if (P[m] >= x) b = m; else a = m + 1;
  }
  return a;
}

// One CTA of 1024: every target's window of sample ranks (nearest rank ceil(p ns) among the ns
// sampled keys, +- dmul sqrt(rank) + dadd) as fixed bins, merged per quantity into sorted
// disjoint intervals, exact-count slots for their bins and a gap index for every other bin;
// counters zeroed.  A plan that does not fit (more than kIvQ intervals or kSpSlots bins) sets
// `fail` with every bin in gap 0: the pass still runs, the check reports a miss.
__global__ void __launch_bounds__(1024) sel_plan_sampled(SampPlan* __restrict__ sp,
                                                       const uint32_t* __restrict__ shist, PctArg pct,
                                                       uint32_t npct, double dmul, double dadd) {
  pdl_wait();  // launched with programmatic stream serialization after its producer (one rank)
  __shared__ unsigned long long pre[2][kFxBins];
  __shared__ unsigned long long part[32 + 1024];
  __shared__ uint32_t tb1[kMaxT], tb2[kMaxT];
  __shared__ uint32_t s_b1[2][kIvQ], s_b2[2][kIvQ], s_slot0[2][kIvQ], s_niv[2];
  const int tid = threadIdx.x;
  auto stamp = [&](int i) {
    if (tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      sp->stamp[i] = t;
    }
  };
  stamp(0);
  for (uint32_t w = 0; w < 2; w++) scan_bins(shist + w * kFxBins, 0ull, w, pre[w], part);
  stamp(1);
  if (tid < (int)(2 * npct)) {
    const uint32_t w = tid >= (int)npct;
    const unsigned long long* P = pre[w];
    const unsigned long long vs = shist[w * kFxBins + (w == 0 ? kFxBins - 2 : 0)];
    const unsigned long long total = P[kFxBins - 1], ns = total + vs;
    uint32_t b1 = 1, b2 = 0;  // empty
    if (ns > 0 && total > 0) {
      const double r = ceil(pct.p[tid % npct] * (double)ns);
      const double ks = r < 1.0 ? 1.0 : (r > (double)ns ? (double)ns : r);
      const double d = dmul * sqrt(ks) + dadd;
      // sample ranks among the counted keys: the single-valued bin sits first (gain == 0) or
      // last (perf == 1) in key order
      const double off = w == 1 ? (double)vs : 0.0;
      const double s_lo = fmax(1.0, floor(ks - d - off)), s_hi = fmax(1.0, ceil(ks + d - off));
      b1 = first_reaching(P, (unsigned long long)fmin(s_lo, (double)total));
      b2 = first_reaching(P, (unsigned long long)fmin(s_hi, (double)total));
    }
    tb1[tid] = b1;
    tb2[tid] = b2;
  }
  __syncthreads();
  stamp(2);
  // per quantity: the targets' non-empty intervals sorted by (b1, target) by a parallel rank
  // count, then merged (overlapping / adjacent) by one thread over the sorted shared arrays
  __shared__ uint32_t srt1[kMaxT], srt2[kMaxT], s_n[2];
  if (tid < 2) s_n[tid] = 0;
  __syncthreads();
  if (tid < (int)(2 * npct)) {
    const uint32_t w = tid >= (int)npct, base = w * npct;
    if (tb1[tid] <= tb2[tid]) {
      uint32_t r = 0;
      for (uint32_t j = base; j < base + npct; j++)
        r += tb1[j] <= tb2[j] && (tb1[j] < tb1[tid] || (tb1[j] == tb1[tid] && j < (uint32_t)tid));
      srt1[base + r] = tb1[tid];
      srt2[base + r] = tb2[tid];
      atomicAdd(&s_n[w], 1u);
    }
  }
  __syncthreads();
  if (tid < 2) {  // thread w merges quantity w
    const uint32_t w = tid, base = w * npct, n = s_n[w];
    uint32_t m = 0, slots = 0, fail = 0;
    for (uint32_t a = 0; a < n && !fail; a++) {
      const uint32_t b1 = srt1[base + a], b2 = srt2[base + a];
      if (m > 0 && b1 <= s_b2[w][m - 1] + 1) {
        if (b2 > s_b2[w][m - 1]) s_b2[w][m - 1] = b2;
      } else if (m == kIvQ) {
        fail = 1;
      } else {
        s_b1[w][m] = b1;
        s_b2[w][m] = b2;
        m++;
      }
    }
    for (uint32_t r = 0; r < m; r++) {
      s_slot0[w][r] = slots;
      slots += s_b2[w][r] - s_b1[w][r] + 1;
    }
    if (slots > kSpSlots) fail = 1;
    s_niv[w] = m;
    sp->nslot[w] = slots;
    s_n[w] = fail;  // reused: this quantity's plan failed
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t fail = s_n[0] | s_n[1];
    if (fail) s_niv[0] = s_niv[1] = 0;  // every bin in gap 0
    sp->fail = fail;
  }
  __syncthreads();
  if (tid < 2 * (int)kIvQ) {
    const uint32_t w = tid / kIvQ, r = tid % kIvQ;
    if (r < s_niv[w]) {
      sp->b1[w][r] = s_b1[w][r];
      sp->b2[w][r] = s_b2[w][r];
      sp->slot0[w][r] = s_slot0[w][r];
    }
    if (r == 0) {
      sp->niv[w] = s_niv[w];
      sp->ncopy[w] = 0;
      sp->ncopy_all[w] = 0;
    }
  }
  stamp(3);
  // per fixed bin: its slot, or its gap = the number of intervals entirely below it; branch-free
  // over the (sorted, disjoint) intervals of its quantity (the early-exit loop of dependent
  // shared loads took ~3.7 us)
  for (uint32_t i = tid; i < 2 * kFxBins; i += blockDim.x) {
    const uint32_t w = i / kFxBins, b = i % kFxBins, niv = s_niv[w];
    uint32_t below = 0, slot = 0xFFFFFFFFu;
#pragma unroll
    for (uint32_t r = 0; r < (uint32_t)kIvQ; r++) {
      const bool v = r < niv;
      const uint32_t b1 = s_b1[w][r], b2 = s_b2[w][r];
      below += (v && b > b2) ? 1u : 0u;
      if (v && b >= b1 && b <= b2) slot = s_slot0[w][r] + b - b1;
    }
    sp->map[w][b] = (uint16_t)(slot != 0xFFFFFFFFu ? (kSpSlotFlag | slot) : below);
  }
  for (uint32_t i = tid; i < 2 * kSpCnt; i += blockDim.x) (&sp->cnt[0][0])[i] = 0;
  __syncthreads();
  stamp(4);
}

// One pass over this rank's keys (kU per quantity in flight per thread, full tiles without
// bounds checks, the tail tile with them): each counted key adds 1 to its slot or gap and the
// slot keys are copied.  Per key: the fixed bin from the key's high word, one shared map
// lookup (uncounted keys read an extra "none" entry).  Gaps (most keys): per-lane 8-bit
// counters packed in registers (gaps 0-7 in a u64, 8-9 in a u32), flushed to shared memory
// every 31 tiles (<= 248 keys per field); slots: one shared atomic per key; copies: a per-warp
// shared stage flushed 32 keys at a time with one reservation.  Per-thread shared gap counters
// instead of the packed registers: 96 M instead of 102 M warp instructions, same time (157-161
// us at 10^9 rows, profiles/r02_sel_pass_gaps_ab.txt): the pass is latency, not issue, bound.
constexpr uint16_t kSpNone = 0x4000u;  // map entry of an uncounted key
#ifndef SP_PIPE
#define SP_PIPE 0  // 1: the next tile's loads in flight while a tile is counted (A/B)
#endif
#ifndef SP_MINB
#define SP_MINB 3  // resident CTAs ptxas budgets registers for (1 / 3 / 4 measured: 1.34 / 1.33 / 1.33 ms reduce + selection at 10^9 rows, pass 177 / 157 / 221 us under ncu)
#endif
template <int kT>
__global__ void __launch_bounds__(kT, SP_MINB) sel_pass_sampled(const double* __restrict__ perf,
                                                       const double* __restrict__ gain, uint64_t lo,
                                                       uint64_t hi, SampPlan* __restrict__ sp,
                                                       double* __restrict__ cbuf) {
  pdl_wait();  // launched with programmatic stream serialization after its producer (one rank)
  constexpr int kU = 8, kFlushTiles = 7;
  static_assert(kFlushTiles * kU < 64, "6-bit gap fields");
  // per fixed bin (+ an entry for uncounted keys) one word: the slot flag in bit 63, else the
  // gap's increment 1 << 6 g (ten 6-bit fields: one 64-bit add counts a key)
  __shared__ uint64_t incm[2][kFxBins + 1];
  __shared__ uint32_t cnt[2][kIvQ + 1];  // gap counters (slots: sel_slot_counts)
  __shared__ uint64_t stage[kT / 32][2][kSpStage];
  for (uint32_t i = threadIdx.x; i < 2 * (kFxBins + 1); i += kT) {
    const uint32_t w = i / (kFxBins + 1), b = i % (kFxBins + 1);
    const uint32_t e = b < kFxBins ? sp->map[w][b] : kSpNone;
    incm[w][b] = (e & kSpSlotFlag) ? (1ull << 63) : (e < 10u ? 1ull << (6 * e) : 0ull);
  }
  if (threadIdx.x < 2 * (kIvQ + 1)) (&cnt[0][0])[threadIdx.x] = 0;
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t gacc[2] = {0ull, 0ull};
  uint32_t nst[2] = {0u, 0u};
  auto flush_gaps = [&]() {
#pragma unroll
    for (int w = 0; w < 2; w++) {
#pragma unroll
      for (int g = 0; g < 10; g++) {
        const uint32_t c = (uint32_t)(gacc[w] >> (6 * g)) & 63u;
        if (c) atomicAdd(&cnt[w][g], c);
      }
      gacc[w] = 0ull;
    }
  };
  auto flush_stage = [&](uint32_t w) {  // warp-collective: every staged key, one reservation
    const uint64_t* sw = stage[wid][w];
    __syncwarp();
    unsigned long long base = 0;
    if (lane == 0) {
      base = atomicAdd(&sp->ncopy[w], (unsigned long long)nst[w]);
      atomicAdd(&sp->ncopy_all[w], (unsigned long long)nst[w]);
    }
    base = __shfl_sync(FULL, base, 0);
    for (uint32_t i = lane; i < nst[w]; i += 32)
      if (base + i < kCompactCap) reinterpret_cast<uint64_t*>(cbuf)[(size_t)w * kCompactCap + base + i] = sw[i];
    __syncwarp();
    nst[w] = 0;
  };
  // per key: slot / gap counts; returns whether the key is copied
  auto count = [&](int w, uint64_t k) -> uint32_t {
    const uint32_t kh = (uint32_t)(k >> 32);  // bins from the high word (32-bit arithmetic)
    uint32_t b;
    if (w == 0)  // perf < 1 (NaN keys are above)
      b = kh < (uint32_t)(kPerfOne >> 32) ? fx_perf_bin_hi(kh) : kFxBins;
    else         // 0 < gain (no gain is below 2^-32 but 0), not NaN
      b = kh - 1u < 0x7FEFFFFFu ? fx_gain_bin_hi(kh) : kFxBins;
    const uint64_t v = incm[w][b];
    gacc[w] += v & ((1ull << 60) - 1);
    // a slot key is only copied: the slot counts are the copies' histogram (sel_slot_counts)
    return (uint32_t)(v >> 63);
  };
  // per tile and quantity: the lanes' copied keys (bit u of mask: key u) placed by one warp
  // scan, staged (or, above the stage, written with their own reservation)
  auto copy_tile = [&](int w, uint32_t mask, const uint64_t* v) {
    const uint32_t c = __popc(mask);
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t total = __shfl_sync(FULL, inc, 31);
    if (total == 0) return;
    if (nst[w] + total > kSpStage) flush_stage(w);
    uint32_t pos = inc - c;
    if (total > kSpStage) {  // more than a stage in one tile: straight out
      unsigned long long base = 0;
      if (lane == 0) {
        base = atomicAdd(&sp->ncopy[w], (unsigned long long)total);
        atomicAdd(&sp->ncopy_all[w], (unsigned long long)total);
      }
      base = __shfl_sync(FULL, base, 0);
#pragma unroll
      for (int u = 0; u < kU; u++)
        if ((mask >> u) & 1u) {
          if (base + pos < kCompactCap) reinterpret_cast<uint64_t*>(cbuf)[(size_t)w * kCompactCap + base + pos] = v[u];
          pos++;
        }
      return;
    }
    pos += nst[w];
#pragma unroll
    for (int u = 0; u < kU; u++)
      if ((mask >> u) & 1u) stage[wid][w][pos++] = v[u];
    nst[w] += total;
    if (nst[w] >= 32) flush_stage(w);
  };
  const uint64_t* P = reinterpret_cast<const uint64_t*>(perf) + lo;
  const uint64_t* Q = reinterpret_cast<const uint64_t*>(gain) + lo;
  const uint64_t n = hi - lo, full = n / (kT * kU);
  int since = 0;
#if SP_PIPE
  // software pipeline: the next tile's loads are issued before this tile is counted
  uint64_t np_[kU], ng_[kU];
  if (blockIdx.x < full) {
    const uint64_t off = blockIdx.x * (uint64_t)(kT * kU) + threadIdx.x;
#pragma unroll
    for (int u = 0; u < kU; u++) {
      np_[u] = __ldcs(P + off + u * kT);
      ng_[u] = __ldcs(Q + off + u * kT);
    }
  }
#endif
  for (uint64_t t = blockIdx.x; t < full; t += gridDim.x) {
    uint64_t vp[kU], vg[kU];
#if SP_PIPE
#pragma unroll
    for (int u = 0; u < kU; u++) {
      vp[u] = np_[u];
      vg[u] = ng_[u];
    }
    if (t + gridDim.x < full) {
      const uint64_t off = (t + gridDim.x) * (kT * kU) + threadIdx.x;
#pragma unroll
      for (int u = 0; u < kU; u++) {
        np_[u] = __ldcs(P + off + u * kT);
        ng_[u] = __ldcs(Q + off + u * kT);
      }
    }
#else
    const uint64_t off = t * (kT * kU) + threadIdx.x;
#pragma unroll
    for (int u = 0; u < kU; u++) {
      vp[u] = __ldcs(P + off + u * kT);
      vg[u] = __ldcs(Q + off + u * kT);
    }
#endif
    uint32_t mp = 0, mg = 0;
#pragma unroll
    for (int u = 0; u < kU; u++) {
      mp |= count(0, vp[u]) << u;
      mg |= count(1, vg[u]) << u;
    }
    copy_tile(0, mp, vp);
    copy_tile(1, mg, vg);
    if (++since == kFlushTiles) {
      flush_gaps();
      since = 0;
    }
  }
  flush_gaps();
  if (blockIdx.x == gridDim.x - 1) {  // the tail tile
    const uint64_t off = full * (kT * kU) + threadIdx.x;
    uint64_t vp[kU], vg[kU];
    uint32_t mp = 0, mg = 0;
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const uint64_t i = off + u * kT;
      vp[u] = i < n ? __ldcs(P + i) : kNaNKey;
      vg[u] = i < n ? __ldcs(Q + i) : kNaNKey;
      mp |= count(0, vp[u]) << u;
      mg |= count(1, vg[u]) << u;
    }
    copy_tile(0, mp, vp);
    copy_tile(1, mg, vg);
  }
  flush_gaps();
#pragma unroll
  for (uint32_t w = 0; w < 2; w++)
    if (nst[w]) flush_stage(w);
  __syncthreads();
  if (threadIdx.x < 2 * (kIvQ + 1)) {
    const uint32_t w = threadIdx.x / (kIvQ + 1), g = threadIdx.x % (kIvQ + 1);
    if (cnt[w][g]) atomicAdd(&sp->cnt[w][kSpSlots + g], cnt[w][g]);
  }
}

// After the pass: the exact count of every slot is the histogram of the copies (every key of
// a slot bin was copied; a copy overflow is caught by the check), per CTA in shared memory,
// flushed once.  Cheaper than a shared atomic per slot key inside the pass (measured: the
// pass 162 -> 142 us at 10^9 rows without them).
__global__ void __launch_bounds__(256) sel_slot_counts(const double* __restrict__ cbuf, SampPlan* __restrict__ sp) {
  pdl_wait();  // launched with programmatic stream serialization after its producer (one rank)
  __shared__ uint16_t map[2][kFxBins];
  __shared__ uint32_t h[2][kSpSlots];
  for (uint32_t i = threadIdx.x; i < 2 * kFxBins; i += blockDim.x) (&map[0][0])[i] = (&sp->map[0][0])[i];
  for (uint32_t i = threadIdx.x; i < 2 * kSpSlots; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
#pragma unroll 1
  for (uint32_t w = 0; w < 2; w++) {
    const uint64_t n = min(sp->ncopy[w], (unsigned long long)kCompactCap);
    const uint64_t* src = reinterpret_cast<const uint64_t*>(cbuf) + (size_t)w * kCompactCap;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += 4 * T) {
      uint64_t k[4];
#pragma unroll
      for (int u = 0; u < 4; u++) k[u] = i + u * T < n ? __ldcg(src + i + u * T) : kNaNKey;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const uint32_t kh = (uint32_t)(k[u] >> 32);
        if (kh >= 0x7FF00000u) continue;  // padding
        const uint32_t e = map[w][w == 0 ? fx_perf_bin_hi(kh) : fx_gain_bin_hi(kh)];
        if (e & kSpSlotFlag) atomicAdd(&h[w][e & (kSpSlotFlag - 1)], 1u);
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 2 * kSpSlots; i += blockDim.x)
    if ((&h[0][0])[i]) atomicAdd(&sp->cnt[i / kSpSlots][i % kSpSlots], (&h[0][0])[i]);
}

// One CTA of 1024, after the pass (its counts summed over ranks): targets from the exact n_def (sel_init's ranks, R-13),
// each target located among the exact counts in key order.  Per quantity the counts form the
// sequence gap 0, interval 0's slots, gap 1, ..., gap niv, plus the single-valued bin (the
// reducer's perf_hist[nb]: perf == 1 is the largest key, gain == 0 the smallest; the plan's
// windows never contain it, so it sits after the last gap resp. before gap 0).  A block scan of
// the sequence, then every target binary-searches its rank.  Inside a slot: narrowed to that
// fixed bin, whose keys all sit in the copies (the state sel_check_sampled leaves); in a gap, a
// total that differs from n_def, an unexpected plan or overflowing copies: sampled_fail (the
// host runs the full selection).
constexpr uint32_t kSpSeq = kSpCnt + 1;  // slots + gaps + the single-valued bin
static_assert(kSpSeq <= 2048, "two elements per thread in the check's scan");
__global__ void __launch_bounds__(1024) sel_check_sampled(SelState* st, const SampPlan* __restrict__ sp,
                                                        const uint64_t* __restrict__ partials, uint32_t nb,
                                                        const uint64_t* __restrict__ mm, PctArg pct,
                                                        uint32_t npct, uint32_t cap, uint32_t force_miss) {
  pdl_wait();  // launched with programmatic stream serialization after its producer (one rank)
  __shared__ unsigned long long pre[2][2048];
  __shared__ uint16_t sbin[2][2048];  // bin of a slot / the single-valued bin; 0xFFFF: a gap
  __shared__ unsigned long long wsum[32];
  __shared__ uint32_t s_fail, s_len[2];
  __shared__ uint32_t q_niv[2], q_nslot[2], q_b1[2][kIvQ], q_slot0[2][kIvQ];  // the plan, in smem
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  const uint64_t n_def = partials[LSCAT_P_RATIO_DEFINED];
  const unsigned long long n_one = partials[LSCAT_P_NCOUNTERS + nb];  // perf == 1 <=> gain == 0
  if (tid < 2 * (int)kIvQ) {
    const uint32_t w = tid / kIvQ, r = tid % kIvQ;
    q_b1[w][r] = sp->b1[w][r];
    q_slot0[w][r] = sp->slot0[w][r];
    if (r == 0) {
      q_niv[w] = sp->niv[w];
      q_nslot[w] = sp->nslot[w];
    }
  }
  if (tid == 0) {
    s_fail = force_miss || sp->fail || sp->ncopy_all[0] > kCompactCap || sp->ncopy_all[1] > kCompactCap;
    for (uint32_t w = 0; w < 2; w++) {
      s_len[w] = sp->nslot[w] + sp->niv[w] + 2;
      // the single-valued bin must lie in the end gap (it never enters a sample window)
      const uint32_t ve = sp->map[w][w == 0 ? kFxBins - 2 : 0];
      if ((ve & kSpSlotFlag) || ve != (w == 0 ? sp->niv[w] : 0u)) s_fail = 1;
    }
  }
  __syncthreads();
  for (uint32_t w = 0; w < 2; w++) {
    // element e of the sequence -> count and bin (gain: the single-valued bin first)
    const uint32_t niv = q_niv[w], len = s_len[w];
    for (uint32_t e = tid; e < 2048; e += blockDim.x) {
      unsigned long long c = 0;
      uint32_t bin = 0xFFFFu;
      if (e < len) {
        const uint32_t q = w == 1 ? e : (e + 1 == len ? 0xFFFFFFFFu : e + 1);  // position after the gain bin
        if (w == 1 ? e == 0 : e + 1 == len) {
          c = n_one;
          bin = w == 0 ? kFxBins - 2 : 0;
        } else {
          // q - 1 = position in gap 0, slots..., gap niv; interval iv's slots start at slot0 + iv + 1
          const uint32_t x = q - 1;
          uint32_t iv = 0;
          while (iv < niv && x >= q_slot0[w][iv] + iv + 1) iv++;
          // x in [slot0[iv-1] + iv, slot0[iv] + iv]: gap iv sits at slot0[iv] + iv (or the end)
          const uint32_t gpos = iv < niv ? q_slot0[w][iv] + iv : q_nslot[w] + niv;
          if (x == gpos) {
            c = sp->cnt[w][kSpSlots + iv];
          } else {  // a slot of interval iv - 1
            const uint32_t r = iv - 1, sl = x - r - 1;
            c = sp->cnt[w][sl];
            bin = q_b1[w][r] + (sl - q_slot0[w][r]);
          }
        }
      }
      pre[w][e] = c;
      sbin[w][e] = (uint16_t)bin;
    }
  }
  __syncthreads();
  for (uint32_t w = 0; w < 2; w++) {  // inclusive scan of 2048 elements, two per thread
    const unsigned long long a0 = pre[w][2 * tid], a1 = pre[w][2 * tid + 1];
    unsigned long long inc = a0 + a1;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      unsigned long long x = wsum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
      }
      wsum[lane] = x;
    }
    __syncthreads();
    const unsigned long long ex = inc - a0 - a1 + (wid ? wsum[wid - 1] : 0ull);
    pre[w][2 * tid] = ex + a0;
    pre[w][2 * tid + 1] = ex + a0 + a1;
    __syncthreads();
  }
  if (tid == 0) {
    st->nt = 2 * npct;
    st->err = 0;
    st->done_ctas = 0;
    st->src = 0;
    st->compact = 0;
    st->n_def = n_def;
    st->sampled_fail = 0;
    st->r0_valid = 0;
    st->nr = 0;
    st->open = 0;
    if (pre[0][2047] != n_def || pre[1][2047] != n_def) s_fail = 1;  // every key counted once
  }
  __syncthreads();
  if (tid < (int)(2 * npct)) {
    Tgt t{};
    t.which = tid >= (int)npct;
    const double r = ceil(pct.p[tid % npct] * (double)n_def);  // nearest rank (R-13)
    t.k = r < 1.0 ? 1 : (r > (double)n_def ? n_def : (uint64_t)r);
    t.done = n_def == 0;
    t.key = kNaNKey;
    t.lo = mm[2 * t.which];
    t.hi = mm[2 * t.which + 1];
    t.count = n_def;
    if (!s_fail && !t.done) {
      const uint32_t w = t.which;
      const unsigned long long* P = pre[w];
      uint32_t lo = 0, hi = 2047;  // smallest e with P[e] >= k
      while (lo < hi) {
        const uint32_t m = (lo + hi) / 2;
        if (P[m] >= t.k) hi = m; else lo = m + 1;
      }
      const uint32_t bin = sbin[w][lo];
      if (bin == 0xFFFFu) {
        atomicOr(&s_fail, 1u);  // inside a gap: a sampling miss
      } else {
        const unsigned long long below = lo ? P[lo - 1] : 0ull;
        uint64_t blo, bhi;
        fx_bin_range(w, bin, &blo, &bhi);
        t.lo = blo > mm[2 * w] ? blo : mm[2 * w];
        t.hi = bhi < mm[2 * w + 1] ? bhi : mm[2 * w + 1];
        t.k -= below;
        t.count = P[lo] - below;
      }
    }
    st->t[tid] = t;
  }
  __syncthreads();
  if (s_fail) {
    if (tid == 0) {
      st->sampled_fail = 1;
      st->nr = 0;
      st->open = 0;
    }
    return;
  }
  if (tid == 0) {
    st->src = 1;  // the later passes read the copies
    st->nc[0] = sp->ncopy[0];
    st->nc[1] = sp->ncopy[1];
  }
  __syncthreads();
  plan_ranges(st, cap);
}

// ---- small inputs on one rank: the whole selection in one cooperative launch ------------
// <= 2^20 keys per quantity (configs[2]/[3] have 0.07 / 0.16 M): the multi-kernel chain above
// is latency bound (~7 dependent launches of 7-20 us each).  One cooperative kernel (one CTA
// per SM, grid-wide barriers between the phases) does: level 0 (the same 8192-bin histogram
// per quantity over [min, max], privatised per CTA), CTA 0 narrows every target to its bin,
// a gather of the keys in those bins, one CTA per bin sorts them and picks the targets.  A bin
// with more than kSmallCap keys sets `fail` and the host runs the chain instead.
constexpr uint32_t kSmallCap = 8192;  // keys per bin selected by one CTA (64 KB of smem)
constexpr uint32_t kRankCountMax = 128;  // phase 4: rank counting up to this many keys

struct SmallSel {
  // results first: the host copies back only this head
  uint64_t tkey[kMaxT];                // per target: result key
  uint32_t fail, nr;
  uint64_t stamp[8];                   // %globaltimer at the phase boundaries (CTA 0; debug)
  // working state
  uint32_t hist[2][kBins];             // level-0 histograms (atomics from every CTA)
  unsigned long long rcnt[kMaxT];      // keys gathered per range
  uint64_t tk[kMaxT];                  // per target: rank inside its range
  uint32_t trange[kMaxT], tdone[kMaxT];
};
constexpr size_t kSmallHead = offsetof(SmallSel, hist);

__global__ void __launch_bounds__(1024, 1) sel_small(const double* __restrict__ perf,
                                                     const double* __restrict__ gain, uint64_t lo,
                                                     uint64_t hi, const uint64_t* __restrict__ partials,
                                                     const uint64_t* __restrict__ mm, PctArg pct,
                                                     uint32_t npct, SmallSel* __restrict__ ss,
                                                     unsigned long long* __restrict__ cand) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned long long dsm[];  // 64 KB: histograms (u32), prefix (u32), sort (u64)
  uint32_t* sh = reinterpret_cast<uint32_t*>(dsm);
  __shared__ uint32_t wsum[32], wsum2[32];
  __shared__ uint64_t s_lo[kMaxT], s_hi[kMaxT], s_k[kMaxT];
  __shared__ uint32_t s_done[kMaxT], s_first[kMaxT], s_range[kMaxT];
  __shared__ uint64_t r_lo[kMaxT], r_hi[kMaxT];
  __shared__ uint32_t r_w[kMaxT], s_nr, s_fail;
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned FULL = 0xffffffffu;
  const uint64_t n_def = partials[LSCAT_P_RATIO_DEFINED];
  const uint32_t nt = 2 * npct;
  Range R[2];
  for (uint32_t w = 0; w < 2; w++) R[w] = make_range(mm[2 * w], mm[2 * w + 1], n_def, w, kSmallCap);
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  auto stamp = [&](int i) {
    if (blockIdx.x == 0 && tid == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ss->stamp[i] = t;
    }
  };
  stamp(0);
  // phase 1: level-0 histograms, privatised per CTA (a gather range needs none)
  for (uint32_t i = tid; i < 2 * kBins; i += blockDim.x) sh[i] = 0;
  if (tid == 0) s_fail = 0;
  __syncthreads();
  for (uint64_t g = lo + blockIdx.x * (uint64_t)blockDim.x + tid; g < hi; g += T) {
#pragma unroll
    for (int w = 0; w < 2; w++) {
      const uint64_t k = (uint64_t)__double_as_longlong((w ? gain : perf)[g]);
      const uint64_t d = k - R[w].lo;
      if (!R[w].gather && d <= R[w].span) atomicAdd(&sh[w * kBins + bin_of_d(R[w], d)], 1u);
    }
  }
  __syncthreads();
  for (uint32_t i = tid; i < 2 * kBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&ss->hist[0][0] + i, sh[i]);
  grid.sync();
  stamp(1);
  // phase 2 (every CTA, identically): every target to its bin; the distinct bins are the ranges.
  // Both histograms are staged in shared memory with coalesced loads first: the scan's
  // thread-contiguous reads straight from L2 (4-byte lanes at a 32-byte stride) fetched every
  // sector 8 times, 512 KB per CTA (5.8 us of the kernel on configs[3], LSCAT_SEL_DEBUG stamps).
  {
    constexpr int kL = 2 * kBins / 1024;  // 1024 threads (the scans below assume it too)
    uint32_t v[kL];
#pragma unroll
    for (int j = 0; j < kL; j++) v[j] = __ldcg(&ss->hist[0][0] + j * 1024 + tid);  // all in flight
#pragma unroll
    for (int j = 0; j < kL; j++) sh[j * 1024 + tid] = v[j];
  }
  __syncthreads();
  {  // inclusive scans of hist[0] and hist[1] into sh[w * kBins ..], in place, both at once
    constexpr int kPer = kBins / 1024;
    uint32_t c[2][kPer], sum[2] = {0u, 0u}, inc[2];
#pragma unroll
    for (int w = 0; w < 2; w++) {
#pragma unroll
      for (int j = 0; j < kPer; j++) { c[w][j] = sh[w * kBins + tid * kPer + j]; sum[w] += c[w][j]; }
      inc[w] = sum[w];
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y0 = __shfl_up_sync(FULL, inc[0], o), y1 = __shfl_up_sync(FULL, inc[1], o);
      if (lane >= o) { inc[0] += y0; inc[1] += y1; }
    }
    if (lane == 31) { wsum[tid >> 5] = inc[0]; wsum2[tid >> 5] = inc[1]; }
    __syncthreads();
    if (tid < 32) {
      uint32_t x0 = wsum[tid], x1 = wsum2[tid];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y0 = __shfl_up_sync(FULL, x0, o), y1 = __shfl_up_sync(FULL, x1, o);
        if (tid >= o) { x0 += y0; x1 += y1; }
      }
      wsum[tid] = x0;
      wsum2[tid] = x1;
    }
    __syncthreads();
    uint32_t run0 = inc[0] - sum[0] + ((tid >> 5) ? wsum[(tid >> 5) - 1] : 0u);
    uint32_t run1 = inc[1] - sum[1] + ((tid >> 5) ? wsum2[(tid >> 5) - 1] : 0u);
#pragma unroll
    for (int j = 0; j < kPer; j++) {
      run0 += c[0][j];
      run1 += c[1][j];
      sh[tid * kPer + j] = run0;
      sh[kBins + tid * kPer + j] = run1;
    }
    __syncthreads();
  }
  stamp(3);
  if (nt <= 32) {
    // one warp, lane i = target i: the same bins, distinct (quantity, bin) pairs and range ids
    // (ranks of the first occurrences in target order) as the general path below, from
    // match_any / ballot in registers instead of O(nt^2) shared-memory loops between barriers
    if (tid < 32) {
      const bool act = tid < (int)nt;
      const uint32_t w = act && tid >= (int)npct;
      uint64_t k = 0, tlo = 0, thi = 0;
      uint32_t done = 1;
      bool too_many = false;
      if (act) {
        const Range& Rw = w ? R[1] : R[0];
        const double r = ceil(pct.p[tid % npct] * (double)n_def);  // nearest rank (R-13)
        k = r < 1.0 ? 1 : (r > (double)n_def ? n_def : (uint64_t)r);
        tlo = Rw.lo;
        thi = Rw.hi;
        done = n_def == 0;
        if (!done && !Rw.gather) {
          const uint32_t* P = sh + w * kBins;
          uint32_t a = 0, b = kBins - 1;  // smallest bin with P[bin] >= k
          while (a < b) {
            const uint32_t m = (a + b) / 2;
            if (P[m] >= k) b = m; else a = m + 1;
          }
          const uint32_t below = a ? P[a - 1] : 0u;
          bin_keys(Rw, (int)a, &tlo, &thi);
          too_many = tlo != thi && P[a] - below > kSmallCap;  // too many to sort
          k -= below;
        }
        if (!done && tlo == thi) done = 2;  // a single-valued bin: the key is known
      }
      const bool open = act && !done;
      // lanes that are not open get a class of their own
      const unsigned m = __match_any_sync(FULL, tlo) & __match_any_sync(FULL, thi) &
                         __match_any_sync(FULL, open ? w : 2u + (uint32_t)tid);
      const int src = __ffs(m) - 1;
      const bool first = open && src == tid;
      const unsigned firsts = __ballot_sync(FULL, first);
      const uint32_t fail = __ballot_sync(FULL, too_many) ? 1u : 0u;
      const uint32_t r = open ? (uint32_t)__popc(firsts & ((1u << src) - 1u)) : 0u;
      if (first) { r_w[r] = w; r_lo[r] = tlo; r_hi[r] = thi; }
      if (act) {
        s_lo[tid] = tlo; s_hi[tid] = thi; s_k[tid] = k; s_done[tid] = done;
        s_first[tid] = first;
        s_range[tid] = r;
        if (blockIdx.x == 0) {
          ss->tk[tid] = k;
          ss->tdone[tid] = done;
          ss->tkey[tid] = done == 2 ? tlo : kNaNKey;
          ss->trange[tid] = r;
        }
      }
      if (tid == 0) {
        const uint32_t nr = (uint32_t)__popc(firsts);
        s_fail = fail;
        s_nr = fail ? 0u : nr;
        if (blockIdx.x == 0) {
          ss->nr = nr;
          ss->fail = fail;
        }
      }
    }
  } else {
    if (tid < (int)nt) {
      const uint32_t w = tid >= (int)npct;
      const double r = ceil(pct.p[tid % npct] * (double)n_def);  // nearest rank (R-13)
      uint64_t k = r < 1.0 ? 1 : (r > (double)n_def ? n_def : (uint64_t)r);
      uint64_t tlo = R[w].lo, thi = R[w].hi;
      uint32_t done = n_def == 0;
      if (!done && !R[w].gather) {
        const uint32_t* P = sh + w * kBins;
        uint32_t a = 0, b = kBins - 1;  // smallest bin with P[bin] >= k
        while (a < b) {
          const uint32_t m = (a + b) / 2;
          if (P[m] >= k) b = m; else a = m + 1;
        }
        const uint32_t below = a ? P[a - 1] : 0u;
        bin_keys(R[w], (int)a, &tlo, &thi);
        if (tlo != thi && P[a] - below > kSmallCap) atomicOr(&s_fail, 1u);  // too many to sort
        k -= below;
      }
      if (!done && tlo == thi) done = 2;  // a single-valued bin: the key is known
      s_lo[tid] = tlo; s_hi[tid] = thi; s_k[tid] = k; s_done[tid] = done;
    }
    __syncthreads();
    // distinct (quantity, bin) -> range ids in target order
    if (tid < (int)nt) {
      bool first = !s_done[tid];
      for (int j = 0; j < tid && first; j++)
        if (!s_done[j] && (j >= (int)npct) == (tid >= (int)npct) && s_lo[j] == s_lo[tid] && s_hi[j] == s_hi[tid])
          first = false;
      s_first[tid] = first;
    }
    __syncthreads();
    if (tid < (int)nt) {
      const uint32_t w = tid >= (int)npct;
      uint32_t r = 0, src = tid;
      if (!s_done[tid]) {
        for (int j = 0; j < tid; j++)  // my range's first occurrence
          if (!s_done[j] && (j >= (int)npct) == (bool)w && s_lo[j] == s_lo[tid] && s_hi[j] == s_hi[tid]) { src = j; break; }
        for (uint32_t j = 0; j < src; j++) r += s_first[j];
        if (src == (uint32_t)tid) { r_w[r] = w; r_lo[r] = s_lo[tid]; r_hi[r] = s_hi[tid]; }
      }
      s_range[tid] = r;
      if (blockIdx.x == 0) {
        ss->tk[tid] = s_k[tid];
        ss->tdone[tid] = s_done[tid];
        ss->tkey[tid] = s_done[tid] == 2 ? s_lo[tid] : kNaNKey;
        ss->trange[tid] = r;
      }
    }
    if (tid == 0) {
      uint32_t nr = 0;
      for (uint32_t j = 0; j < nt; j++) nr += s_first[j];
      s_nr = s_fail ? 0u : nr;
      if (blockIdx.x == 0) {
        ss->nr = nr;
        ss->fail = s_fail;
      }
    }
  }
  __syncthreads();
  stamp(4);
  // phase 3: gather the keys of the ranges (disjoint bins: at most one range per key)
  const uint32_t nr = s_nr;
  if (nr) {
    for (uint64_t g0 = lo + blockIdx.x * (uint64_t)blockDim.x; g0 < hi; g0 += T) {
      const uint64_t g = g0 + tid;
#pragma unroll
      for (int w = 0; w < 2; w++) {
        const uint64_t k = g < hi ? (uint64_t)__double_as_longlong((w ? gain : perf)[g]) : kNaNKey;
        uint32_t r = 0xFFFFFFFFu;
        for (uint32_t q = 0; q < nr; q++)
          if (r_w[q] == (uint32_t)w && r_lo[q] <= k && k <= r_hi[q]) r = q;
        const unsigned peers = __match_any_sync(FULL, r);
        const int leader = __ffs(peers) - 1;
        unsigned long long base = 0;
        if (r != 0xFFFFFFFFu && lane == leader) base = atomicAdd(&ss->rcnt[r], (unsigned long long)__popc(peers));
        base = __shfl_sync(FULL, base, leader);
        if (r != 0xFFFFFFFFu) {
          const unsigned long long at = base + __popc(peers & ((1u << lane) - 1u));
          if (at < kSmallCap) cand[(size_t)r * kSmallCap + at] = k;
        }
      }
    }
  }
  stamp(5);
  grid.sync();
  stamp(2);
  // phase 4: CTA r (mod the grid) picks its targets' keys among range r's gathered keys: by
  // rank counting when there are few (one key per thread, O(n^2) compares), else by a radix
  // select in shared memory (8-bit digits of the key below the range's common prefix; one
  // histogram pass per digit and target).  A bitonic sort of up to 8192 keys took ~20 us and
  // rank counting at n = 1024 as long (issue bound: n compares in every thread).
  __shared__ uint32_t s_dh[256];
  __shared__ unsigned long long s_pre, s_surv[kRankCountMax];
  __shared__ uint64_t s_kk;
  __shared__ uint32_t s_cnt, s_m;
  for (uint32_t r = blockIdx.x; r < nr; r += gridDim.x) {
  const uint32_t n = (uint32_t)min(ss->rcnt[r], (unsigned long long)kSmallCap);
  if (ss->rcnt[r] <= kRankCountMax) {
    for (uint32_t i = tid; i < n; i += blockDim.x) dsm[i] = cand[(size_t)r * kSmallCap + i];
    __syncthreads();
    if (tid < (int)n) {  // my key's rank: smaller keys, and equal keys earlier in the list
      const unsigned long long x = dsm[tid];
      uint32_t rank = 0;
      for (uint32_t j = 0; j < n; j++) {
        const unsigned long long y = dsm[j];
        rank += (y < x) || (y == x && j < (uint32_t)tid);
      }
      for (uint32_t i = 0; i < nt; i++)
        if (!s_done[i] && s_range[i] == r && s_k[i] == rank + 1) ss->tkey[i] = x;
    }
    if (tid < (int)nt && !s_done[tid] && s_range[tid] == r && !(s_k[tid] >= 1 && s_k[tid] <= n))
      atomicOr(&ss->fail, 2u);  // keys lost: the host falls back
  } else {
    for (uint32_t i = tid; i < n; i += blockDim.x) dsm[i] = cand[(size_t)r * kSmallCap + i];
    // every key of the range lies in [r_lo, r_hi]: the digits above their highest differing
    // bit are common
    const uint64_t diff = r_lo[r] ^ r_hi[r];
    const int top = diff ? 64 - __clzll((long long)diff) : 0;  // bits below the common prefix
    for (uint32_t i = 0; i < nt; i++) {  // CTA-uniform loop over the range's targets
      if (s_done[i] || s_range[i] != r) continue;
      const uint64_t k0 = s_k[i];
      if (!(k0 >= 1 && k0 <= n)) {
        if (tid == 0) atomicOr(&ss->fail, 2u);  // keys lost: the host falls back
        continue;
      }
      if (tid == 0) { s_pre = r_lo[r] & ~((top >= 64) ? ~0ull : ((1ull << top) - 1)); s_kk = k0; s_cnt = n; }
      __syncthreads();  // s_cnt is read at the loop head (and the keys are in place)
      // digits until the keys with the chosen prefix are few: those are then ranked directly
      // (after the first digit typically ~n / 256 keys remain; each further digit pass costs
      // three barriers, ~1.4 us)
      int sh_end = 0;
      for (int sh0 = ((top + 7) / 8) * 8 - 8; sh0 >= 0; sh0 -= 8) {
        if (s_cnt <= kRankCountMax) { sh_end = sh0 + 8; break; }  // CTA-uniform
        if (tid < 256) s_dh[tid] = 0;
        __syncthreads();
        const unsigned long long pre = s_pre;
        const unsigned long long hmask = (sh0 + 8 >= 64) ? 0ull : (~0ull << (sh0 + 8));
        // (warp-aggregating these atomics with match.any measured slower: 7.0 -> 7.9 us)
        for (uint32_t j = tid; j < n; j += blockDim.x) {
          const unsigned long long x = dsm[j];
          if ((x & hmask) == (pre & hmask)) atomicAdd(&s_dh[(uint32_t)(x >> sh0) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {  // the digit holding the kk-th of the keys with this prefix
          uint32_t c[8], sum = 0;
#pragma unroll
          for (int q = 0; q < 8; q++) { c[q] = s_dh[tid * 8 + q]; sum += c[q]; }
          uint32_t inc = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
          }
          const uint64_t kk = s_kk;
          const uint32_t ex = inc - sum;
          if (tid == 31 && inc < kk) atomicOr(&ss->fail, 2u);  // keys lost: the host falls back
          if (ex < kk && kk <= inc) {  // exactly one lane
            uint32_t cum = ex;
            int q = 0;
            while (cum + c[q] < kk) cum += c[q++];
            s_pre = (pre & hmask) | ((unsigned long long)(tid * 8 + q) << sh0);
            s_kk = kk - cum;
            s_cnt = c[q];
          }
        }
        __syncthreads();
      }
      if (sh_end == 0) {  // every digit chosen: s_pre is the key
        if (tid == 0) ss->tkey[i] = s_pre;
      } else {  // rank the s_cnt keys with the prefix above bit sh_end
        const unsigned long long pmask = sh_end >= 64 ? 0ull : (~0ull << sh_end);
        const unsigned long long pre = s_pre & pmask;
        if (tid == 0) s_m = 0;
        __syncthreads();
        for (uint32_t j = tid; j < n; j += blockDim.x) {
          const unsigned long long x = dsm[j];
          if ((x & pmask) == pre) {
            const uint32_t at = atomicAdd(&s_m, 1u);
            if (at < kRankCountMax) s_surv[at] = x;
          }
        }
        __syncthreads();
        const uint32_t m = s_m;
        const uint64_t kk = s_kk;
        if (tid == 0 && (m > kRankCountMax || !(kk >= 1 && kk <= m))) atomicOr(&ss->fail, 2u);  // keys lost
        if (tid < (int)m && m <= kRankCountMax) {  // the survivors' order is arbitrary; the value is unique
          const unsigned long long x = s_surv[tid];
          uint32_t rank = 0;
          for (uint32_t j = 0; j < m; j++) {
            const unsigned long long y = s_surv[j];
            rank += (y < x) || (y == x && j < (uint32_t)tid);
          }
          if (rank + 1 == kk) ss->tkey[i] = x;
        }
      }
      __syncthreads();  // s_pre / s_kk / s_cnt / s_surv are reset for the next target
    }
  }
  __syncthreads();  // the next range reuses dsm
  }
  if (tid == 0) {  // debug: the latest CTA end (the launch is preceded by a memset of *ss)
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax((unsigned long long*)&ss->stamp[6], (unsigned long long)t);
  }
}

// Grid of sel_small: one CTA per 512 keys, at most one per SM (tiny inputs get fewer CTAs and
// cheaper grid barriers).  Calibration on configs[2]/[3] (LSCAT_SMALL_KEYS_PER_CTA = 512 / 2048
// / 4096 / 8192 / 16384): reduce + early selection 0.090 / 0.091 / 0.101 / 0.106 / 0.127 ms and
// 0.116 / 0.116 / 0.119 / 0.130 / 0.155 ms (profiles/r02_sel_small_grid.txt): the CTAs' loads
// in flight win over the flush and barrier costs.  Re-checked after the session-3 rework
// (256 / 512 / 1024 / 2048): 71.6-76.5 / 83.0-86.8 us, within the run-to-run spread.
uint32_t small_grid(const lscat_ctx* ctx, uint64_t n) {
  static const uint64_t per = [] {
    const char* e = getenv("LSCAT_SMALL_KEYS_PER_CTA");
    const long long v = e ? atoll(e) : 0;
    return v > 0 ? (uint64_t)v : (uint64_t)512;
  }();
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(ctx->sm_count, (n + per - 1) / per));
}

// ---- after the sampled first level, on one rank: the rest of the selection in one launch ----
// sel_check_sampled leaves every open target in a range [lo, hi] (one fixed bin) whose keys
// all sit in the copies.  The chain would now run ~4 histogram levels over the copies (two
// dependent launches each).  One cooperative kernel does it instead: each range's keys are
// counted into kFinBins sub-bins (global atomics; ranges found by a scan over the <= 18 sorted
// ranges), CTA r narrows range r's targets to their sub-bins, the keys of those
// sub-bins are gathered, one CTA per sub-bin sorts them and picks.  The SelState is only read:
// a sub-bin above kSmallCap keys (or any inconsistency) sets `fail` and the host continues
// with the chain from the unchanged state.
constexpr uint32_t kFinBins = 2048;
constexpr uint32_t kFinRanges = 2 * kIvQ;
constexpr size_t kFinSmem = (size_t)kSmallCap * 8;  // the sort

struct FinSel {
  // results first: the host copies back only this head
  uint64_t tkey[kMaxT];                    // per open target: result key
  uint32_t fail, pad;
  uint64_t stamp[5];                       // %globaltimer at the phase boundaries (CTA 0; debug)
  // working state
  uint64_t tlo[kMaxT], thi[kMaxT], tk[kMaxT], tcnt[kMaxT];  // per target after the narrowing
  unsigned long long rcnt[kMaxT];          // keys gathered per sub-range
  uint32_t hist[kFinRanges][kFinBins];
};
constexpr size_t kFinHead = offsetof(FinSel, tlo);

__global__ void __launch_bounds__(1024, 1) sel_finish(const SelState* __restrict__ st,
                                                      const double* __restrict__ cbuf,
                                                      FinSel* __restrict__ fs,
                                                      unsigned long long* __restrict__ cand,
                                                      uint32_t force_fail) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned long long dsm[];  // the phase-4 sort
  __shared__ uint64_t r_lo[kFinRanges], r_hi[kFinRanges];
  __shared__ uint32_t r_sh[kFinRanges];
  __shared__ uint64_t q_lo[kMaxT], q_hi[kMaxT];  // sub-ranges (gather): key interval, quantity
  __shared__ uint32_t q_w[kMaxT], s_qr[kMaxT], s_first[kMaxT], s_nq;
  __shared__ unsigned long long wsum[32];
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned FULL = 0xffffffffu;
  const uint32_t nr = st->nr, nw0 = st->nw0, nt = st->nt;
  const bool on = !force_fail && !st->sampled_fail && st->src == 1 && st->err == 0 && nr <= kFinRanges;
  if (!on) {
    if (blockIdx.x == 0 && tid == 0) fs->fail = 1;
    return;  // grid-uniform: no grid barrier is reached
  }
  auto stamp = [&](int i) {
    if (blockIdx.x == 0 && tid == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      fs->stamp[i] = t;
    }
  };
  stamp(0);
  if (nr == 0) {  // every target resolved by the check: nothing to do
    if (blockIdx.x == 0 && tid == 0) fs->fail = 0;
    return;
  }
  __shared__ uint64_t s_tk[kMaxT];
  __shared__ uint32_t s_trange[kMaxT], s_topen[kMaxT], s_tw[kMaxT];
  // After the check every range is one fixed bin of selbins.h (clipped to [min, max]): a key's
  // range is found from its fixed bin through a byte map (0xFF: no range)
  __shared__ uint8_t rmap[2 * kFxBins];
  __shared__ uint32_t gbm[kFinRanges][kFinBins / 32];  // phase 3: sub-bins to gather
  __shared__ uint32_t s_bad;
  for (uint32_t i = tid; i < 2 * kFxBins; i += blockDim.x) rmap[i] = 0xFF;
  for (uint32_t i = tid; i < kFinRanges * (kFinBins / 32); i += blockDim.x) (&gbm[0][0])[i] = 0u;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  if (tid < (int)nr) {
    const Range& R = st->r[tid];
    r_lo[tid] = R.lo;
    r_hi[tid] = R.hi;
    const uint64_t span = R.hi - R.lo;
    uint32_t s = 0;
    while ((span >> s) >= kFinBins) s++;
    r_sh[tid] = s;
    const uint32_t w = R.which;
    const uint32_t b = fx_bin(w, R.lo);
    if (b != fx_bin(w, R.hi) || virtual_bin(w, b) || (tid < (int)nw0) != (w == 0)) atomicOr(&s_bad, 1u);
    else rmap[w * kFxBins + b] = (uint8_t)tid;
  }
  if (tid < (int)nt) {  // the targets, read once (phases 2 and 3 loop over them)
    const Tgt& t = st->t[tid];
    s_tk[tid] = t.k;
    s_trange[tid] = t.range;
    s_topen[tid] = !t.done;
    s_tw[tid] = t.which;
  }
  __syncthreads();
  if (s_bad) {  // not one fixed bin per range (never, with the check above): the chain
    if (blockIdx.x == 0 && tid == 0) fs->fail = 16;
    return;  // CTA-uniform and identical in every CTA: no grid barrier is reached
  }
  // phase 1: sub-bin counts of every range (ranges of quantity w: [w ? nw0 : 0, w ? nr : nw0)),
  // straight to the global histogram: the keys spread over nr x kFinBins bins, so a per-CTA
  // privatised copy would cost a flush of ~all its bins per CTA.  kU loads in flight per thread.
  // range of a copied key: its fixed bin's map entry, if the key also lies inside the range's
  // clipped [lo, hi] (copies of a range's bin outside [min, max] do not exist)
  auto i_range = [&](int w, uint64_t k) -> uint32_t {
    const uint32_t kh = (uint32_t)(k >> 32);
    // counted keys only (perf < 1, finite gain): the padding NaN keys have no bin
    if (kh >= (w == 0 ? (uint32_t)(kPerfOne >> 32) : 0x7FF00000u)) return 0xFFu;
    const uint32_t b = w == 0 ? fx_perf_bin_hi(kh) : fx_gain_bin_hi(kh);
    const uint32_t r = rmap[w * kFxBins + b];
    return (r != 0xFFu && r_lo[r] <= k && k <= r_hi[r]) ? r : 0xFFu;
  };
  constexpr int kU = 8;
  const uint64_t* keys = reinterpret_cast<const uint64_t*>(cbuf);
  const uint64_t cstride = (uint64_t)gridDim.x * blockDim.x * kU;
#pragma unroll 1
  for (int w = 0; w < 2; w++) {
    const uint32_t a = w ? nw0 : 0, b = w ? nr : nw0;
    if (a == b) continue;
    const uint64_t n = min(st->nc[w], (unsigned long long)kCompactCap);
    const uint64_t* src = keys + (size_t)w * kCompactCap;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * kU + tid; base < n; base += cstride) {
      uint64_t k[kU];
#pragma unroll
      for (int u = 0; u < kU; u++) {
        const uint64_t i = base + (uint64_t)u * blockDim.x;
        k[u] = i < n ? __ldcg(src + i) : kNaNKey;
      }
#pragma unroll
      for (int u = 0; u < kU; u++) {
        const uint32_t r = i_range(w, k[u]);
        if (r != 0xFFu) atomicAdd(&fs->hist[r][(uint32_t)((k[u] - r_lo[r]) >> r_sh[r])], 1u);
      }
    }
  }
  grid.sync();
  stamp(1);
  // phase 2: CTA r narrows range r's open targets to their sub-bins
  if (blockIdx.x < nr) {
    const uint32_t r = blockIdx.x;
    constexpr int kPer = kFinBins / 1024;
    uint32_t c[kPer];
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < kPer; j++) { c[j] = __ldcg(&fs->hist[r][tid * kPer + j]); sum += c[j]; }
    unsigned long long inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[tid >> 5] = inc;
    __syncthreads();
    if (tid < 32) {
      unsigned long long x = wsum[tid];
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL, x, o);
        if (tid >= o) x += y;
      }
      wsum[tid] = x;
    }
    __syncthreads();
    const unsigned long long ex = inc - sum + ((tid >> 5) ? wsum[(tid >> 5) - 1] : 0ull);
    if (tid == 1023 && ex + sum != st->r[r].count) atomicOr(&fs->fail, 2u);  // keys lost
    for (uint32_t i = 0; i < nt; i++) {
      if (!s_topen[i] || s_trange[i] != r) continue;
      const uint64_t k = s_tk[i];
      if (tid == 1023 && !(k >= 1 && k <= ex + sum)) atomicOr(&fs->fail, 2u);  // rank outside
      if (!(ex < k && k <= ex + sum)) continue;
      unsigned long long cum = ex;
      int j = 0;
      while (cum + c[j] < k) cum += c[j++];
      const uint32_t bb = (uint32_t)(tid * kPer + j);
      const uint64_t lo = r_lo[r] + ((uint64_t)bb << r_sh[r]);
      const uint64_t top = lo + ((1ull << r_sh[r]) - 1);
      const uint64_t hi = (top < lo || top > r_hi[r]) ? r_hi[r] : top;
      fs->tlo[i] = lo;
      fs->thi[i] = hi;
      fs->tk[i] = k - cum;
      fs->tcnt[i] = c[j];
      if (c[j] > kSmallCap && hi != lo) atomicOr(&fs->fail, 4u);  // too many to sort
    }
  }
  grid.sync();
  stamp(2);
  if (__ldcg(&fs->fail)) return;  // grid-uniform (written before the barrier)
  // phase 3 (every CTA, identically): distinct open sub-ranges; gather their keys
  if (nt <= 32) {
    // one warp, lane i = target i: first occurrences and sub-range ids from match_any / ballot
    // (the same values as the general path below, without its O(nt^2) loops between barriers)
    if (tid < 32) {
      const bool act = tid < (int)nt;
      const bool open = act && s_topen[tid];
      const uint64_t lo = open ? __ldcg(&fs->tlo[tid]) : 0ull, hi = open ? __ldcg(&fs->thi[tid]) : 0ull;
      const uint32_t w = act ? s_tw[tid] : 0u;
      const bool cand = open && hi != lo;
      const unsigned m = __match_any_sync(FULL, lo) & __match_any_sync(FULL, hi) &
                         __match_any_sync(FULL, cand ? w : 2u + (uint32_t)tid);
      const int src = __ffs(m) - 1;
      const bool first = cand && src == tid;
      const unsigned firsts = __ballot_sync(FULL, first);
      if (act) {
        q_lo[tid] = lo;
        q_hi[tid] = hi;
        q_w[tid] = w;
        s_first[tid] = first;
        s_qr[tid] = cand ? (uint32_t)__popc(firsts & ((1u << src) - 1u)) : 0xFFFFFFFFu;
      }
      if (tid == 0) s_nq = (uint32_t)__popc(firsts);
    }
    __syncthreads();
  } else {
    if (tid < (int)nt) {
      const bool open = s_topen[tid];
      q_lo[tid] = open ? __ldcg(&fs->tlo[tid]) : 0ull;
      q_hi[tid] = open ? __ldcg(&fs->thi[tid]) : 0ull;
      q_w[tid] = s_tw[tid];
      s_first[tid] = open && q_hi[tid] != q_lo[tid];
    }
    __syncthreads();
    const bool mine_first = tid < (int)nt && s_first[tid];
    bool dup = false;
    if (mine_first)
      for (int j = 0; j < tid; j++)
        if (s_first[j] && q_w[j] == q_w[tid] && q_lo[j] == q_lo[tid] && q_hi[j] == q_hi[tid]) { dup = true; break; }
    __syncthreads();
    if (mine_first && dup) s_first[tid] = 0;
    __syncthreads();
    if (tid < (int)nt) {  // sub-range id of every open target (its first occurrence's rank)
      uint32_t q = 0xFFFFFFFFu;
      if (s_topen[tid] && q_hi[tid] != q_lo[tid]) {
        uint32_t src = tid;
        for (int j = 0; j < tid; j++)
          if (s_first[j] && q_w[j] == q_w[tid] && q_lo[j] == q_lo[tid] && q_hi[j] == q_hi[tid]) { src = j; break; }
        q = 0;
        for (uint32_t j = 0; j < src; j++) q += s_first[j];
      }
      s_qr[tid] = q;
    }
    if (tid == 0) {
      uint32_t n = 0;
      for (uint32_t j = 0; j < nt; j++) n += s_first[j];
      s_nq = n;
    }
    __syncthreads();
  }
  // compact the distinct sub-ranges to the front: sub-range q = the q-th first occurrence
  __shared__ uint64_t g_lo[kMaxT], g_hi[kMaxT];
  __shared__ uint32_t g_w[kMaxT];
  if (tid < (int)nt && s_first[tid]) {
    const uint32_t q = s_qr[tid];
    g_lo[q] = q_lo[tid];
    g_hi[q] = q_hi[tid];
    g_w[q] = q_w[tid];
    const uint32_t r = s_trange[tid];
    const uint32_t sb = (uint32_t)((q_lo[tid] - r_lo[r]) >> r_sh[r]);
    atomicOr(&gbm[r][sb >> 5], 1u << (sb & 31));
  }
  __syncthreads();
  const uint32_t nq = s_nq;
#pragma unroll 1
  for (int w = 0; w < 2; w++) {
    const uint64_t n = min(st->nc[w], (unsigned long long)kCompactCap);
    const uint64_t* src = keys + (size_t)w * kCompactCap;
    // CTA-uniform trip count (the warp collectives below): every thread runs every chunk
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * kU; base < n; base += cstride) {
      uint64_t k[kU];
#pragma unroll
      for (int u = 0; u < kU; u++) {
        const uint64_t i = base + (uint64_t)u * blockDim.x + tid;
        k[u] = i < n ? __ldcg(src + i) : kNaNKey;
      }
#pragma unroll
      for (int u = 0; u < kU; u++) {
        const uint32_t r = i_range(w, k[u]);
        bool hit = false;
        if (r != 0xFFu) {
          const uint32_t sb = (uint32_t)((k[u] - r_lo[r]) >> r_sh[r]);
          hit = (gbm[r][sb >> 5] >> (sb & 31)) & 1u;
        }
        if (!__any_sync(FULL, hit)) continue;
        uint32_t q = 0xFFFFFFFFu;
        if (hit)
          for (uint32_t j = 0; j < nq; j++)
            if (g_w[j] == (uint32_t)w && g_lo[j] <= k[u] && k[u] <= g_hi[j]) q = j;
        const unsigned peers = __match_any_sync(FULL, q);
        const int leader = __ffs(peers) - 1;
        unsigned long long at0 = 0;
        if (q != 0xFFFFFFFFu && lane == leader) at0 = atomicAdd(&fs->rcnt[q], (unsigned long long)__popc(peers));
        at0 = __shfl_sync(FULL, at0, leader);
        if (q != 0xFFFFFFFFu) {
          const unsigned long long at = at0 + __popc(peers & ((1u << lane) - 1u));
          if (at < kSmallCap) cand[(size_t)q * kSmallCap + at] = k[u];
        }
      }
    }
  }
  grid.sync();
  stamp(3);
  // phase 4: CTA q sorts sub-range q's keys (bitonic, shared memory) and picks its targets'
  if (blockIdx.x == 0 && tid < (int)nt) {  // single-valued sub-bins: the key is known
    if (s_topen[tid] && q_hi[tid] == q_lo[tid]) fs->tkey[tid] = q_lo[tid];
  }
  if (blockIdx.x >= nq) return;
  const uint32_t q = blockIdx.x;
  const unsigned long long cnt = __ldcg(&fs->rcnt[q]);
  const uint32_t n = (uint32_t)min(cnt, (unsigned long long)kSmallCap);
  uint32_t P2 = 1;
  while (P2 < n) P2 <<= 1;
  for (uint32_t i = tid; i < P2; i += blockDim.x) dsm[i] = i < n ? __ldcg(&cand[(size_t)q * kSmallCap + i]) : ~0ull;
  __syncthreads();
  for (uint32_t kk = 2; kk <= P2; kk <<= 1)
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      for (uint32_t i = tid; i < P2; i += blockDim.x) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = dsm[i], b = dsm[ixj];
          if ((a > b) == ((i & kk) == 0)) { dsm[i] = b; dsm[ixj] = a; }
        }
      }
      __syncthreads();
    }
  if (tid < (int)nt && s_qr[tid] == q) {
    const uint64_t k = __ldcg(&fs->tk[tid]);
    if (cnt == __ldcg(&fs->tcnt[tid]) && k >= 1 && k <= n) fs->tkey[tid] = dsm[k - 1];
    else atomicOr(&fs->fail, 8u);  // keys lost: the host continues with the chain
  }
  stamp(4);
}

PctArg pct_arg(const double* pct, uint32_t npct) {
  PctArg pa{};
  for (uint32_t i = 0; i < npct; i++) pa.p[i] = pct[i];
  return pa;
}

bool coop_supported(lscat_ctx* ctx) {
  int coop = 0;
  return cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device) == cudaSuccess && coop;
}

// Device / pinned buffers of the selection, by scratch name (grow-only, shared by every path).
struct SelBufs {
  SelState* st = nullptr;
  SelState* hst = nullptr;  // pinned
  uint32_t* hist = nullptr;
  unsigned long long* cand = nullptr;
  double* cbuf = nullptr;
  uint32_t* shist = nullptr;
  SampPlan* sp = nullptr;
  FinSel* fs = nullptr;
  FinSel* fsh = nullptr;  // pinned head
  unsigned long long* fcand = nullptr;
};

// One shared-memory carve-out (maximum shared) for every kernel of the selection paths, as for
// the reducer and the level chain: a kernel whose carve-out differs from its predecessor's
// waits for the SMs to be reconfigured (measured at 10^9 rows: the one-CTA plan and check
// kernels took 18 / 16 us between events, mostly that wait).  Once per device.
lscat_status sel_carveout(lscat_ctx* ctx) {
  static std::atomic<bool> done[64] = {};  // ranks of the local transport are threads
  const int d = ctx->device;
  if (d >= 0 && d < 64 && done[d].load(std::memory_order_acquire)) return LSCAT_OK;
  const void* fs[] = {(const void*)sel_sample_hist, (const void*)sel_plan_sampled, (const void*)sel_slot_counts,
                      (const void*)sel_pass_sampled<256>, (const void*)sel_check_sampled,
                      (const void*)sel_finish, (const void*)sel_small};
  for (const void* f : fs)
    LSCAT_CUDA(ctx, cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         (int)cudaSharedmemCarveoutMaxShared));
  if (d >= 0 && d < 64) done[d].store(true, std::memory_order_release);
  return LSCAT_OK;
}

lscat_status sel_bufs(lscat_ctx* ctx, uint32_t cap, SelBufs* b) {
  if (lscat_status cs = sel_carveout(ctx)) return cs;
  cudaError_t err = cudaSuccess;
  auto S = [&](const char* name, size_t bytes) { void* p = scratch(ctx, name, bytes, &err); return p; };
  b->st = (SelState*)S("sel_state", sizeof(SelState));
  if (!err) b->hist = (uint32_t*)S("sel_hist", (size_t)kMaxR * kBins * 4);
  if (!err) b->cand = (unsigned long long*)S("sel_cand", (size_t)kMaxR * (cap + 1) * 8);
  if (!err) b->cbuf = (double*)S("sel_cbuf", 2 * kCompactCap * 8);
  if (!err) b->shist = (uint32_t*)S("sel_shist", 2 * kFxBins * 4);
  if (!err) b->sp = (SampPlan*)S("sel_samp", sizeof(SampPlan));
  if (!err) b->fs = (FinSel*)S("sel_fin", sizeof(FinSel));
  if (!err) b->fcand = (unsigned long long*)S("sel_fin_cand", (size_t)kMaxT * kSmallCap * 8);
  if (err) return cuda_fail(ctx, err, "selection: scratch");
  b->hst = (SelState*)pinned(ctx, "sel_state_h", sizeof(SelState), &err);
  if (!err) b->fsh = (FinSel*)pinned(ctx, "sel_fin_h", kFinHead, &err);
  if (err) return cuda_fail(ctx, err, "selection: pinned");
  return LSCAT_OK;
}

// LSCAT_SEL_TIMING=1 (calibration): CUDA events between the stages of the sampled selection,
// printed once the selection is collected (stderr).  Not used inside graph capture.
std::vector<std::pair<const char*, cudaEvent_t>>& sel_events() {
  static std::vector<std::pair<const char*, cudaEvent_t>> v;
  return v;
}
bool sel_timing_on() {
  static const bool on = getenv("LSCAT_SEL_TIMING") != nullptr;
  return on;
}
void sel_mark(const char* name, cudaStream_t q) {
  if (!sel_timing_on()) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(q, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, q);
  sel_events().push_back({name, e});
}
void sel_print_events() {
  auto& v = sel_events();
  if (v.empty()) return;
  cudaEventSynchronize(v.back().second);
  fprintf(stderr, "sel timing (us):");
  for (size_t i = 1; i < v.size(); i++) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, v[i - 1].second, v[i].second);
    fprintf(stderr, " %s %.1f", v[i].first, ms * 1e3f);
  }
  fprintf(stderr, "\n");
  for (auto& e : v) cudaEventDestroy(e.second);
  v.clear();
}

// The sampled first level on stream q: sample, plan, pass, (NCCL sums,) check.  With `fin`
// (one rank) the state after the check is copied to the host and sel_finish follows
// (launch_finish); else the caller enqueues levels.
lscat_status enqueue_sampled(lscat_ctx* ctx, const SelBufs& B, const double* perf, const double* gain,
                             uint64_t lo, uint64_t hi, const uint64_t* partials, const uint64_t* mm,
                             uint32_t nb, const PctArg& pa, uint32_t npct, uint32_t cap, bool fin,
                             cudaStream_t q) {
  const int world = ctx->world;
  const uint64_t n = hi - lo;
  if (!fin) {  // the chain follows at once (with sel_finish: cleared only if it hands over)
    LSCAT_CUDA(ctx, cudaMemsetAsync(B.hist, 0, (size_t)kMaxR * kBins * 4, q));
    LSCAT_CUDA(ctx, cudaMemsetAsync(B.cand, 0, (size_t)kMaxR * 8, q));
  }
  sel_mark("start", q);
  LSCAT_CUDA(ctx, cudaMemsetAsync(B.shist, 0, 2 * kFxBins * 4, q));
  const uint64_t rstride = std::max<uint64_t>(kSampleRun, n / kSampleRuns);
  const int grid_s = (int)std::min<uint64_t>(kSampleRuns * kSampleRun / 256, (uint64_t)ctx->sm_count * 2);
  sel_sample_hist<<<grid_s, 256, 0, q>>>(perf, gain, lo, hi, rstride, B.shist);
  LSCAT_CUDA(ctx, cudaGetLastError());
  sel_mark("sample", q);
  if (world > 1) {
    lscat_status ns = ctx->comm->allreduce(ctx, {{B.shist, 2 * (size_t)kFxBins, DT::U32, Op::Sum}}, q);
    if (ns) return ns;
  }
  const bool pdl = world == 1 && !sel_timing_on();  // (stage events between the kernels: plain launches)
  LSCAT_CUDA(ctx, launch_pdl(sel_plan_sampled, dim3(1), dim3(1024), 0, q, pdl, B.sp, B.shist, pa, npct, 4.5, 32.0));
  sel_mark("plan", q);
  static const int occ_p = [] {  // resident CTAs per SM of the pass (binary property; one-time)
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, sel_pass_sampled<256>, 256, 0);
    cudaGetLastError();
    return std::max(v, 1);
  }();
  const int grid_p = (int)std::min<uint64_t>(std::max<uint64_t>(1, (n + 256 * 8 - 1) / (256 * 8)),
                                             (uint64_t)ctx->sm_count * occ_p);
  LSCAT_CUDA(ctx, launch_pdl(sel_pass_sampled<256>, dim3(grid_p), dim3(256), 0, q, pdl, perf, gain, lo, hi, B.sp, B.cbuf));
  sel_mark("pass", q);
  LSCAT_CUDA(ctx, launch_pdl(sel_slot_counts, dim3(ctx->sm_count * 4), dim3(256), 0, q, pdl,  // 4 CTAs per SM
                             B.cbuf, B.sp));
  sel_mark("slots", q);
  if (world > 1) {  // exact counts and copy totals over all ranks
    lscat_status ns = ctx->comm->allreduce(ctx, {{&B.sp->cnt[0][0], 2 * (size_t)kSpCnt, DT::U32, Op::Sum},
                                                 {&B.sp->ncopy_all[0], 2, DT::U64, Op::Sum}}, q);
    if (ns) return ns;
  }
  // LSCAT_SEL_FORCE_MISS=1 (tests): every sampled first level reports a miss
  static const uint32_t force_miss = getenv("LSCAT_SEL_FORCE_MISS") != nullptr ? 1u : 0u;
  LSCAT_CUDA(ctx, launch_pdl(sel_check_sampled, dim3(1), dim3(1024), 0, q, pdl && world == 1, B.st, B.sp, partials,
                             nb, mm, pa, npct, cap, force_miss));
  sel_mark("check", q);
  if (fin) {  // sel_finish follows; the state as the check left it
    LSCAT_CUDA(ctx, cudaMemsetAsync(B.fs, 0, sizeof(FinSel), q));
    LSCAT_CUDA(ctx, cudaMemcpyAsync(B.hst, B.st, sizeof(SelState), cudaMemcpyDeviceToHost, q));
  }
  return LSCAT_OK;
}

// One rank, after enqueue_sampled(fin): the rest of the selection in one cooperative launch;
// its result head is copied to the host.
lscat_status launch_finish(lscat_ctx* ctx, const SelBufs& B, cudaStream_t q) {
  LSCAT_CUDA(ctx, ensure_smem_attr((const void*)sel_finish, kFinSmem));
  // LSCAT_SEL_FIN_FORCE_FAIL=1 (tests): sel_finish hands over to the chain at once
  static const uint32_t ff = getenv("LSCAT_SEL_FIN_FORCE_FAIL") != nullptr ? 1u : 0u;
  const SelState* st_c = B.st;
  const double* cb_c = B.cbuf;
  FinSel* fs = B.fs;
  unsigned long long* fc = B.fcand;
  uint32_t ff_ = ff;
  void* args[] = {(void*)&st_c, (void*)&cb_c, (void*)&fs, (void*)&fc, (void*)&ff_};
  LSCAT_CUDA(ctx, cudaLaunchCooperativeKernel((const void*)sel_finish, dim3(ctx->sm_count), dim3(1024), args,
                                              kFinSmem, q));
  sel_mark("finish", q);
  LSCAT_CUDA(ctx, cudaMemcpyAsync(B.fsh, B.fs, kFinHead, cudaMemcpyDeviceToHost, q));
  ctx->launches++;
  return LSCAT_OK;
}

}  // namespace

lscat_status early_select(lscat_ctx* ctx, const double* perf, const double* gain, uint64_t lo, uint64_t hi,
                          const uint64_t* partials, const uint64_t* mm, uint32_t nb, const double* pct,
                          uint32_t npct, cudaStream_t s, uint32_t* kind) {
  static_assert(kEarlySmallGroups == kSmallKeys, "small-table threshold");
  *kind = EARLY_NONE;
  if (ctx->world != 1 || !coop_supported(ctx) || hi <= lo) return LSCAT_OK;
  static const bool no_small = getenv("LSCAT_SEL_NOSMALL") != nullptr;
  static const bool no_sample = getenv("LSCAT_SEL_NOSAMPLE") != nullptr;
  static const bool no_finish = getenv("LSCAT_SEL_NOFINISH") != nullptr;
  if (lscat_status cs = sel_carveout(ctx)) return cs;
  const PctArg pa = pct_arg(pct, npct);
  cudaError_t err;
  if (hi - lo <= kSmallKeys) {  // the one-launch selection
    if (no_small) return LSCAT_OK;
    SmallSel* sm = (SmallSel*)scratch(ctx, "sel_small", sizeof(SmallSel), &err);
    if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
    auto* scand = (unsigned long long*)scratch(ctx, "sel_small_cand", (size_t)kMaxT * kSmallCap * 8, &err);
    if (err) return cuda_fail(ctx, err, "reduce_table: scratch");
    SmallSel* hsm = (SmallSel*)pinned(ctx, "sel_small_h", sizeof(SmallSel), &err);
    if (err) return cuda_fail(ctx, err, "reduce_table: pinned");
    constexpr size_t kSmallSmem = (size_t)kSmallCap * 8;
    LSCAT_CUDA(ctx, ensure_smem_attr((const void*)sel_small, kSmallSmem));
    LSCAT_CUDA(ctx, cudaMemsetAsync(sm, 0, sizeof(SmallSel), s));
    void* args[] = {(void*)&perf, (void*)&gain, (void*)&lo, (void*)&hi, (void*)&partials,
                    (void*)&mm, (void*)&pa, (void*)&npct, (void*)&sm, (void*)&scand};
    LSCAT_CUDA(ctx, cudaLaunchCooperativeKernel((const void*)sel_small, dim3(small_grid(ctx, hi - lo)), dim3(1024),
                                                args, kSmallSmem, s));
    ctx->launches++;
    LSCAT_CUDA(ctx, cudaMemcpyAsync(hsm, sm, kSmallHead, cudaMemcpyDeviceToHost, s));
    *kind = EARLY_SMALL;
    return LSCAT_OK;
  }
  if (npct > (uint32_t)kIvQ || no_sample || no_finish) return LSCAT_OK;
  SelBufs B;
  lscat_status bs = sel_bufs(ctx, 8192, &B);
  if (bs) return bs;
  if ((bs = enqueue_sampled(ctx, B, perf, gain, lo, hi, partials, mm, nb, pa, npct, 8192, true, s))) return bs;
  ctx->launches += 5;
  if ((bs = launch_finish(ctx, B, s))) return bs;
  *kind = EARLY_SAMPLED;
  return LSCAT_OK;
}

namespace {

lscat_status select_percentiles(lscat_ctx* ctx, const double* pct, uint32_t npct, double* out_perf,
                                double* out_gain, cudaStream_t s) {
  const ReduceState& rs = ctx->rs;
  const int world = ctx->world;
  const uint32_t cap = world > 1 ? 1024 : 8192;
  const size_t cand_len = (size_t)kMaxR * (cap + 1);
  cudaError_t err;
  SelBufs B;
  if (lscat_status bs = sel_bufs(ctx, cap, &B)) return bs;
  SelState* st = B.st;
  uint32_t* hist = B.hist;
  unsigned long long* cand = B.cand;
  unsigned long long* cand_all = cand;
  if (world > 1) {
    cand_all = (unsigned long long*)scratch(ctx, "sel_cand_all", (size_t)world * cand_len * 8, &err);
    if (err) return cuda_fail(ctx, err, "stats: scratch");
  }
  double* cbuf = B.cbuf;
  SelState* hst = B.hst;
  constexpr int kT0 = 512, kT1 = 256;
  const int pass_smem = kSmemRanges * kBins * 4, res_smem = (int)cap * 8;
  // kernel attributes and occupancy: once per process (per resolve smem size)
  int& occ0 = ctx->sel_occ0;
  int& occ1 = ctx->sel_occ1;
  LSCAT_CUDA(ctx, ensure_smem_attr((const void*)sel_pass<true, kT0>, pass_smem));
  LSCAT_CUDA(ctx, ensure_smem_attr((const void*)sel_resolve, res_smem));
  if (!occ0) {
    LSCAT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, sel_pass<true, kT0>, kT0, pass_smem));
    LSCAT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, sel_pass<false, kT1>, kT1, 0));
    occ0 = std::max(occ0, 1);
    occ1 = std::max(occ1, 1);
    // one shared-memory carve-out for the whole chain: a kernel whose carve-out differs from
    // its predecessor's waits for the SMs to be reconfigured (measured: ~18 us of a 20 us
    // sel_resolve on a small table was launch, not work)
    const void* chain[] = {(const void*)sel_init, (const void*)sel_pass<true, kT0>,
                           (const void*)sel_pass<false, kT1>, (const void*)sel_pass<false, kT1, 1>,
                           (const void*)sel_resolve};
    for (const void* f : chain)
      LSCAT_CUDA(ctx, cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           (int)cudaSharedmemCarveoutMaxShared));
  }
  // grids: every resident CTA once (occupancy API), capped by the work (kU x 32 groups per warp)
  const uint64_t n = rs.own_hi - rs.own_lo;
  const int grid0 = (int)std::min<uint64_t>(std::max<uint64_t>(1, (n + kT0 * 8 - 1) / (kT0 * 8)),
                                             (uint64_t)ctx->sm_count * occ0);
  const bool small = n <= kSmallKeys;
  const int grid1 = small ? (int)std::min<uint64_t>(std::max<uint64_t>(1, (n + kT1 - 1) / kT1),
                                                    (uint64_t)ctx->sm_count * occ1)
                          : (int)std::min<uint64_t>(std::max<uint64_t>(1, (n + kT1 * 8 - 1) / (kT1 * 8)),
                                                    (uint64_t)ctx->sm_count * occ1);
  const int lpb = small ? kLevelsPerBatchSmall : kLevelsPerBatch;
  PctArg pa{};
  for (uint32_t i = 0; i < npct; i++) pa.p[i] = pct[i];
  // R-27: lscat_reduce_table already enqueued the selection of these percentiles
  const bool early_match = rs.early != EARLY_NONE && rs.early_pct.size() == npct &&
                           std::equal(rs.early_pct.begin(), rs.early_pct.end(), pct);
  const bool early_sm = early_match && rs.early == EARLY_SMALL;
  const bool early_samp = early_match && rs.early == EARLY_SAMPLED;
  // any other selection reuses the state buffers the early result sits in
  if (!early_match) ctx->rs.early = EARLY_NONE;
  static const bool dbg_early = getenv("LSCAT_SEL_DEBUG") != nullptr;
  if (dbg_early && early_match) fprintf(stderr, "sel early %s\n", early_sm ? "small" : "sampled");
  if (early_sm) {  // the one-launch selection ran right after the reducer
    SmallSel* hsm = (SmallSel*)pinned(ctx, "sel_small_h", sizeof(SmallSel), &err);
    if (err) return cuda_fail(ctx, err, "stats: pinned");
    LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
    if (dbg_early)
      fprintf(stderr, "sel early small: fail %u nr %u phases(ns) %lld %lld (scan %lld targets %lld gather %lld barrier %lld)\n",
              hsm->fail, hsm->nr, (long long)(hsm->stamp[1] - hsm->stamp[0]), (long long)(hsm->stamp[2] - hsm->stamp[1]),
              (long long)(hsm->stamp[3] - hsm->stamp[1]), (long long)(hsm->stamp[4] - hsm->stamp[3]),
              (long long)(hsm->stamp[5] - hsm->stamp[4]), (long long)(hsm->stamp[2] - hsm->stamp[5]));
    if (dbg_early)
      fprintf(stderr, "  prologue->stamp0 n/a, phase 4 (to the last CTA's end) %lld ns\n",
              (long long)(hsm->stamp[6] - hsm->stamp[2]));
    if (dbg_early) {  // keys per range (the working state after the head: a separate copy)
      std::vector<SmallSel> full(1);
      const SmallSel* smd = (const SmallSel*)scratch(ctx, "sel_small", sizeof(SmallSel), &err);
      if (!err && cudaMemcpy(full.data(), smd, sizeof(SmallSel), cudaMemcpyDeviceToHost) == cudaSuccess)
        for (uint32_t r = 0; r < hsm->nr && r < kMaxT; r++) fprintf(stderr, "  range %u keys %llu\n", r, full[0].rcnt[r]);
    }
    if (!hsm->fail) {
      for (uint32_t i = 0; i < 2 * npct; i++) {
        double v;
        memcpy(&v, &hsm->tkey[i], 8);
        (i >= npct ? out_gain : out_perf)[i % npct] = v;
      }
      return LSCAT_OK;
    }
    ctx->sel_fallbacks++;  // a bin too large for one CTA: the chain below
    ctx->rs.early = EARLY_NONE;
  }
  static const bool no_small = getenv("LSCAT_SEL_NOSMALL") != nullptr;
  if (small && world == 1 && !no_small && !early_sm && npct <= kMaxT / 2) {  // one cooperative launch
    int coop = 0;
    LSCAT_CUDA(ctx, cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device));
    constexpr size_t kSmallSmem = (size_t)kSmallCap * 8;  // >= 2 x kBins x 4
    static_assert(kSmallSmem >= 2 * kBins * 4, "sel_small shared memory");
    if (coop) {
      SmallSel* sm = (SmallSel*)scratch(ctx, "sel_small", sizeof(SmallSel), &err);
      if (err) return cuda_fail(ctx, err, "stats: scratch");
      auto* scand = (unsigned long long*)scratch(ctx, "sel_small_cand", (size_t)kMaxT * kSmallCap * 8, &err);
      if (err) return cuda_fail(ctx, err, "stats: scratch");
      SmallSel* hsm = (SmallSel*)pinned(ctx, "sel_small_h", sizeof(SmallSel), &err);
      if (err) return cuda_fail(ctx, err, "stats: pinned");
      LSCAT_CUDA(ctx, ensure_smem_attr((const void*)sel_small, kSmallSmem));
      LSCAT_CUDA(ctx, cudaMemsetAsync(sm, 0, sizeof(SmallSel), s));
      const double* perf_p = rs.perf;
      const double* gain_p = rs.gain;
      uint64_t lo_ = rs.own_lo, hi_ = rs.own_hi;
      const uint64_t* part_p = rs.partials;
      const uint64_t* mm_p = rs.minmax;
      uint32_t np_ = npct;
      void* args[] = {(void*)&perf_p, (void*)&gain_p, (void*)&lo_, (void*)&hi_, (void*)&part_p,
                      (void*)&mm_p, (void*)&pa, (void*)&np_, (void*)&sm, (void*)&scand};
      LSCAT_CUDA(ctx, cudaLaunchCooperativeKernel((const void*)sel_small, dim3(small_grid(ctx, rs.own_hi - rs.own_lo)),
                                                  dim3(1024), args, kSmallSmem, s));
      ctx->launches++;
      const bool dbg = getenv("LSCAT_SEL_DEBUG") != nullptr;
      LSCAT_CUDA(ctx, cudaMemcpyAsync(hsm, sm, dbg ? sizeof(SmallSel) : kSmallHead, cudaMemcpyDeviceToHost, s));
      LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
      if (dbg) {
        fprintf(stderr, "sel_small: fail %u nr %u phases(ns) %lld %lld\n", hsm->fail, hsm->nr,
                (long long)(hsm->stamp[1] - hsm->stamp[0]), (long long)(hsm->stamp[2] - hsm->stamp[1]));
        for (uint32_t r = 0; r < hsm->nr && r < kMaxT; r++) fprintf(stderr, "  range %u keys %llu\n", r, hsm->rcnt[r]);
        for (uint32_t i = 0; i < 2 * npct; i++)
          fprintf(stderr, "  t%u done %u range %u k %llu key %016llx\n", i, hsm->tdone[i], hsm->trange[i],
                  (unsigned long long)hsm->tk[i], (unsigned long long)hsm->tkey[i]);
      }
      if (!hsm->fail) {
        for (uint32_t i = 0; i < 2 * npct; i++) {
          double v;
          memcpy(&v, &hsm->tkey[i], 8);
          (i >= npct ? out_gain : out_perf)[i % npct] = v;
        }
        return LSCAT_OK;
      }
      ctx->sel_fallbacks++;  // a bin too large for one CTA: the multi-kernel chain below
    }
  }
  // One batch: lpb levels of pass -> (merge) -> resolve -> plan, then the state
  // is read back (one host sync per batch).
  auto enqueue_levels = [&](cudaStream_t q, bool first) -> lscat_status {
    for (int level = 0; level < lpb; level++) {
      if (first && level == 0)
        sel_pass<true, kT0><<<grid0, kT0, pass_smem, q>>>(rs.perf, rs.gain, rs.own_lo, rs.own_hi, st, hist, cand, cap, cbuf);
      else
        if (small)
          sel_pass<false, kT1, 1><<<grid1, kT1, 0, q>>>(rs.perf, rs.gain, rs.own_lo, rs.own_hi, st, hist, cand, cap, cbuf);
        else
          sel_pass<false, kT1><<<grid1, kT1, 0, q>>>(rs.perf, rs.gain, rs.own_lo, rs.own_hi, st, hist, cand, cap, cbuf);
      LSCAT_CUDA(ctx, cudaGetLastError());
      if (world > 1) {
        lscat_status ns = ctx->comm->allreduce(ctx, {{hist, (size_t)kMaxR * kBins, DT::U32, Op::Sum}}, q);
        if (ns) return ns;
        ns = ctx->comm->allgather(ctx, cand, cand_all, cand_len, DT::U64, q);
        if (ns) return ns;
      }
      // one CTA per open range: at most one range per open target
      sel_resolve<<<std::min<int>(kMaxR, 2 * (int)npct), 1024, res_smem, q>>>(st, hist, cand_all, cand, world, cap);
      LSCAT_CUDA(ctx, cudaGetLastError());
    }
    LSCAT_CUDA(ctx, cudaMemcpyAsync(hst, st, sizeof(SelState), cudaMemcpyDeviceToHost, q));
    return LSCAT_OK;
  };
  // sampled first level (large inputs, <= kIvQ percentiles; LSCAT_SEL_NOSAMPLE=1 disables it)
  static const bool no_sample = getenv("LSCAT_SEL_NOSAMPLE") != nullptr;
  bool sampled = early_samp || (!small && npct <= (uint32_t)kIvQ && !no_sample);
  // one rank: the levels after the sampled first level run as one cooperative sel_finish
  // (LSCAT_SEL_NOFINISH=1 keeps the chain)
  static const bool no_finish = getenv("LSCAT_SEL_NOFINISH") != nullptr;
  const bool fin = early_samp || (sampled && world == 1 && !no_finish && coop_supported(ctx));
  FinSel* fsh = B.fsh;
  auto enqueue_first_sampled = [&](cudaStream_t q) -> lscat_status {
    lscat_status es = enqueue_sampled(ctx, B, rs.perf, rs.gain, rs.own_lo, rs.own_hi, rs.partials, rs.minmax,
                                      rs.opts.bins_per_unit, pa, npct, cap, fin, q);
    if (es || fin) return es;  // sel_finish follows (outside the graph)
    return enqueue_levels(q, false);
  };
  auto enqueue_first = [&](cudaStream_t q) -> lscat_status {
    LSCAT_CUDA(ctx, cudaMemsetAsync(hist, 0, (size_t)kMaxR * kBins * 4, q));
    LSCAT_CUDA(ctx, cudaMemsetAsync(cand, 0, (size_t)kMaxR * 8, q));
    sel_init<<<1, kMaxT, 0, q>>>(st, rs.partials, rs.minmax, pa, npct, cap);
    LSCAT_CUDA(ctx, cudaGetLastError());
    return enqueue_levels(q, true);
  };
  const bool debug = getenv("LSCAT_SEL_DEBUG") != nullptr;
  lscat_status ls;
  // First batch: launched as a cached CUDA graph when the selection runs on one rank (the
  // small tables of configs[2]/[3] are launch-latency bound: ~10 dependent launches).
  auto launch_first = [&](bool samp) -> lscat_status {
    auto enq = [&](cudaStream_t q) { return samp ? enqueue_first_sampled(q) : enqueue_first(q); };
    if (world == 1 && !debug) {
      std::string key;
      auto put = [&](const void* v, size_t n_) { key.append(reinterpret_cast<const char*>(v), n_); };
      const void* ptrs[] = {rs.perf, rs.gain, rs.partials, rs.minmax, st, hist, cand, cbuf, hst, B.sp, B.shist};
      put(ptrs, sizeof ptrs);
      put(&rs.own_lo, 8); put(&rs.own_hi, 8); put(&npct, 4); put(pa.p, npct * 8);
      put(&grid0, 4); put(&grid1, 4); put(&cap, 4); put(&samp, sizeof samp);
      const bool fin_k = samp && fin;
      put(&fin_k, sizeof fin_k); put(&B.fs, sizeof B.fs);
      cudaGraphExec_t gx = nullptr;
      for (auto& kv : ctx->sel_graphs)
        if (kv.first == key) gx = kv.second;
      if (!gx) {
        cudaStream_t cs = ctx->capture_stream;
        LSCAT_CUDA(ctx, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        lscat_status e = enq(cs);
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(cs, &g);
        if (e) {
          if (g) cudaGraphDestroy(g);
          return e;
        }
        LSCAT_CUDA(ctx, ce);
        const cudaError_t ie = cudaGraphInstantiate(&gx, g, 0);
        cudaGraphDestroy(g);
        LSCAT_CUDA(ctx, ie);
        if (ctx->sel_graphs.size() >= 8) {  // small LRU-less cache: drop the oldest
          cudaGraphExecDestroy(ctx->sel_graphs.front().second);
          ctx->sel_graphs.erase(ctx->sel_graphs.begin());
        }
        ctx->sel_graphs.emplace_back(std::move(key), gx);
      }
      LSCAT_CUDA(ctx, cudaGraphLaunch(gx, s));
    } else {
      lscat_status e = enq(s);
      if (e) return e;
    }
    if (samp && fin) {
      if (lscat_status fe = launch_finish(ctx, B, s)) return fe;
      ctx->launches += 5;
    } else {
      ctx->launches += (samp ? 5 : 1) + 2 * lpb;
    }
    return LSCAT_OK;
  };
  if (!early_samp)
    if ((ls = launch_first(sampled))) return ls;
  bool levels_pending = sampled && fin;  // the first batch ran no levels (sel_finish instead)
  bool chain_cleared = !(sampled && fin);  // the sampled path with sel_finish skips the chain's memsets
  for (int batch = 0;; batch++) {
    if (batch == 8) return fail(ctx, LSCAT_ERR_STATE, "stats: percentile selection did not converge");
    if (batch > 0) {
      if (!chain_cleared) {  // sel_finish handed over: the chain's histograms / counters first
        LSCAT_CUDA(ctx, cudaMemsetAsync(hist, 0, (size_t)kMaxR * kBins * 4, s));
        LSCAT_CUDA(ctx, cudaMemsetAsync(cand, 0, (size_t)kMaxR * 8, s));
        chain_cleared = true;
      }
      if ((ls = enqueue_levels(s, false))) return ls;
      ctx->launches += 2 * lpb;
    }
    LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
    if (batch == 0 && sampled) sel_print_events();
    if (debug && batch == 0 && sampled) {  // the sampled plan and its exact counts
      std::vector<SampPlan> h(1);
      LSCAT_CUDA(ctx, cudaMemcpy(h.data(), B.sp, sizeof(SampPlan), cudaMemcpyDeviceToHost));
      const SampPlan& f = h[0];
      for (uint32_t w = 0; w < 2; w++) {
        unsigned long long sum = 0;
        for (uint32_t i = 0; i < kSpCnt; i++) sum += f.cnt[w][i];
        if (w == 0)
          fprintf(stderr, "plan phases(ns): scans %lld targets %lld merge %lld map %lld\n",
                  (long long)(f.stamp[1] - f.stamp[0]), (long long)(f.stamp[2] - f.stamp[1]),
                  (long long)(f.stamp[3] - f.stamp[2]), (long long)(f.stamp[4] - f.stamp[3]));
        fprintf(stderr, "samp q%u: fail %u niv %u nslot %u ncopy %llu counted %llu intervals", w, f.fail,
                f.niv[w], f.nslot[w], f.ncopy[w], sum);
        for (uint32_t r = 0; r < f.niv[w]; r++) fprintf(stderr, " [%u,%u]", f.b1[w][r], f.b2[w][r]);
        fprintf(stderr, "\n");
      }
    }
    if (debug)
      fprintf(stderr, "sel batch %d: nt %u nr %u nw0 %u open %u err %u src %u compact %u nc %llu %llu sampled %d fail %u\n",
              batch, hst->nt, hst->nr, hst->nw0, hst->open, hst->err, hst->src, hst->compact, hst->nc[0],
              hst->nc[1], (int)sampled, hst->sampled_fail);
    if (batch == 0 && levels_pending && !hst->sampled_fail) {
      levels_pending = false;
      if (debug)
        fprintf(stderr, "sel_finish: fail %u open %u nr %u nc %llu %llu phases(ns) %lld %lld %lld %lld\n",
                fsh->fail, hst->open, hst->nr, hst->nc[0], hst->nc[1],
                (long long)(fsh->stamp[1] - fsh->stamp[0]), (long long)(fsh->stamp[2] - fsh->stamp[1]),
                (long long)(fsh->stamp[3] - fsh->stamp[2]), (long long)(fsh->stamp[4] - fsh->stamp[3]));
      if (!fsh->fail && !hst->err) {
        for (uint32_t i = 0; i < 2 * npct; i++) {
          const Tgt& t = hst->t[i];
          const uint64_t key = t.done ? t.key : fsh->tkey[i];
          double v;
          memcpy(&v, &key, 8);
          (t.which ? out_gain : out_perf)[i % npct] = v;
        }
        return LSCAT_OK;
      }
      ctx->fin_fallbacks++;  // the chain continues from the state the check left
      if (hst->err) return fail(ctx, LSCAT_ERR_STATE, "stats: percentile selection lost keys (code %u)", hst->err);
      if (!hst->open) break;
      continue;
    }
    if (batch == 0 && sampled && hst->sampled_fail) {  // a sampling miss: the histogram path
      sampled = false;
      levels_pending = false;
      ctx->sel_fallbacks++;
      ctx->rs.early = EARLY_NONE;
      if ((ls = launch_first(false))) return ls;
      batch = -1;
      continue;
    }
    if (hst->err) return fail(ctx, LSCAT_ERR_STATE, "stats: percentile selection lost keys (code %u)", hst->err);
    if (!hst->open) break;
  }
  for (uint32_t i = 0; i < 2 * npct; i++) {
    const Tgt& t = hst->t[i];
    double v;
    memcpy(&v, &t.key, 8);
    (t.which ? out_gain : out_perf)[i % npct] = v;
  }
  return LSCAT_OK;
}

}  // namespace
}  // namespace lscat

using namespace lscat;

extern "C" lscat_status lscat_stats(lscat_ctx* ctx, const lscat_reduce_opts* o, lscat_stats_out* out,
                                    void* stream) {
  LSCAT_CHECK_CTX(ctx);
  if (!o || !out) return fail(ctx, LSCAT_ERR_INVALID_ARG, "stats: null argument");
  const ReduceState& rs = ctx->rs;
  if (!rs.valid) return fail(ctx, LSCAT_ERR_STATE, "stats: call lscat_reduce_table first");
  if (memcmp(&rs.opts, o, sizeof *o) != 0)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "stats: options differ from the last reduce_table");
  if (out->n_percentiles > 64 || (out->n_percentiles && (!out->percentiles || !out->pct_perf || !out->pct_gain)))
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "stats: bad percentile arguments");
  for (uint32_t i = 0; i < out->n_percentiles; i++)
    if (!(out->percentiles[i] >= 0.0 && out->percentiles[i] <= 1.0))
      return fail(ctx, LSCAT_ERR_INVALID_ARG, "stats: percentile %u outside [0, 1]", i);
  if (out->n_percentiles && (!rs.perf || !rs.gain))
    return fail(ctx, LSCAT_ERR_STATE, "stats: percentiles need keep_values or caller perf/gain arrays");
  cudaStream_t s = (cudaStream_t)stream;
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));
  const size_t nb = o->bins_per_unit, ng = (size_t)o->gain_cap * nb, nbb = (size_t)o->n_matrices * o->n_blocks;
  const size_t plen = LSCAT_P_NCOUNTERS + (nb + 1) + (ng + 1) + nbb * (o->block_profile ? 3 : 1) +
                      (o->kernel_rollup ? 8 + nb + 1 : 0);
  cudaError_t err;
  // the reduce call already enqueued the host copy when it enqueued the one-launch selection
  // for exactly these percentiles (rs.partials_h; same buffer, same length)
  const bool pre_copied = rs.partials_h && rs.early == EARLY_SMALL && out->n_percentiles &&
                          rs.early_pct.size() == out->n_percentiles &&
                          memcmp(rs.early_pct.data(), out->percentiles, out->n_percentiles * 8) == 0;
  uint64_t* hP = (uint64_t*)pinned(ctx, "stats_partials", plen * 8, &err);
  if (err) return cuda_fail(ctx, err, "stats: pinned");
  if (!pre_copied || hP != rs.partials_h)
    LSCAT_CUDA(ctx, cudaMemcpyAsync(hP, rs.partials, plen * 8, cudaMemcpyDeviceToHost, s));
  if (out->n_percentiles) {
    // a8 on the device; its first host sync also completes the partials copy above
    lscat_status st = select_percentiles(ctx, out->percentiles, out->n_percentiles, out->pct_perf,
                                         out->pct_gain, s);
    if (st) return st;
  } else {
    LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  }
  std::vector<uint64_t> P(hP, hP + plen);
  const uint64_t* C = P.data();
  if (C[LSCAT_P_BAD_IDS])
    return fail(ctx, LSCAT_ERR_INVALID_ARG,
                "stats: %llu groups of the reduced table have a block_id >= n_blocks or a matrix "
                "index >= n_matrices", (unsigned long long)C[LSCAT_P_BAD_IDS]);
  out->n_rows = C[LSCAT_P_ROWS]; out->n_ok = C[LSCAT_P_OK]; out->n_nan = C[LSCAT_P_NAN];
  out->n_invalid = C[LSCAT_P_INVALID]; out->n_groups = C[LSCAT_P_GROUPS];
  out->n_defined = C[LSCAT_P_DEFINED]; out->n_all_nan = C[LSCAT_P_ALL_NAN];
  out->n_complete = C[LSCAT_P_COMPLETE]; out->n_incomplete = C[LSCAT_P_INCOMPLETE];
  out->n_largest_missing = C[LSCAT_P_LARGEST_MISSING]; out->n_ratio_defined = C[LSCAT_P_RATIO_DEFINED];
  out->n_largest_is_best = C[LSCAT_P_LARGEST_IS_BEST];
  out->n_largest_strictly_slower = C[LSCAT_P_LARGEST_SLOWER];
  out->n_gain_gt = C[LSCAT_P_GAIN_GT]; out->n_perf_lt = C[LSCAT_P_PERF_LT]; out->n_perf_band = C[LSCAT_P_PERF_BAND];
  out->perf_fx_hi = C[LSCAT_P_PERF_FX_HI]; out->perf_fx_lo = C[LSCAT_P_PERF_FX_LO];
  out->gain_fx_hi = C[LSCAT_P_GAIN_FX_HI]; out->gain_fx_lo = C[LSCAT_P_GAIN_FX_LO];
  // a10: fractions and exact fixed-point means (O3 steps 9 and 11)
  const double nrd = (double)out->n_ratio_defined;
  out->frac_nonnan = out->n_rows ? (double)out->n_ok / (double)out->n_rows : NAN;
  out->frac_largest_not_best = nrd > 0 ? (double)(out->n_ratio_defined - out->n_largest_is_best) / nrd : NAN;
  out->frac_gain_gt = nrd > 0 ? (double)out->n_gain_gt / nrd : NAN;
  out->frac_perf_lt = nrd > 0 ? (double)out->n_perf_lt / nrd : NAN;
  out->frac_perf_band = nrd > 0 ? (double)out->n_perf_band / nrd : NAN;
  const unsigned __int128 tp = ((unsigned __int128)out->perf_fx_hi << 21) + out->perf_fx_lo;
  const unsigned __int128 tgn = ((unsigned __int128)out->gain_fx_hi << 21) + out->gain_fx_lo;
  out->mean_perf = nrd > 0 ? ((double)tp * 0x1p-52) / nrd : NAN;
  out->mean_gain = nrd > 0 ? ((double)tgn * 0x1p-32) / nrd : NAN;
  const uint64_t* H = C + LSCAT_P_NCOUNTERS;
  if (out->perf_hist) memcpy(out->perf_hist, H, (nb + 1) * 8);
  if (out->gain_hist) memcpy(out->gain_hist, H + nb + 1, (ng + 1) * 8);
  if (out->best_block_hist) memcpy(out->best_block_hist, H + nb + 1 + ng + 1, nbb * 8);
  if (o->kernel_rollup) {  // R-26: the per-kernel roll-up
    const uint64_t* K = C + plen - (8 + nb + 1);
    out->n_kernels = K[0];
    out->n_kernels_largest_not_best = K[1];
    out->n_kernels_perf_lt = K[2];
    out->n_kernels_perf_band = K[3];
    out->kernel_mean_fx_hi = K[4];
    out->kernel_mean_fx_lo = K[5];
    const double nk = (double)K[0];
    out->frac_kernels_largest_not_best = K[0] ? (double)K[1] / nk : NAN;
    out->frac_kernels_perf_lt = K[0] ? (double)K[2] / nk : NAN;
    out->frac_kernels_perf_band = K[0] ? (double)K[3] / nk : NAN;
    const unsigned __int128 tk = ((unsigned __int128)K[4] << 21) + K[5];
    out->mean_kernel_perf = K[0] ? ((double)tk * 0x1p-52) / nk : NAN;
    if (out->kernel_perf_hist) memcpy(out->kernel_perf_hist, K + 8, (nb + 1) * 8);
  }
  if (o->block_profile) {  // R-22: mean of best / r_b per (matrix, block)
    const uint64_t* ps = H + nb + 1 + ng + 1 + nbb;
    const uint64_t* pc = ps + nbb;
    for (size_t i = 0; i < nbb; i++) {
      if (out->profile_count) out->profile_count[i] = pc[i];
      if (out->profile_mean) out->profile_mean[i] = pc[i] ? ((double)ps[i] * 0x1p-31) / (double)pc[i] : NAN;
    }
  }
  return LSCAT_OK;
}
