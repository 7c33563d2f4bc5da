// stats.cu — a10 (finalize the merged integer partials on the host) and a8 (exact
// nearest-rank percentiles of perf and gain over ratio-defined groups, R-13).
//
// Percentile selection is a multi-level radix select over the IEEE bit patterns of the
// positive doubles (bit order == value order): a level splits a key range [lo, hi] into
// 4096 bins (bin 0 = {lo}, last bin = {hi}, the rest partition (lo, hi) by a shift), one pass
// over the keys builds the histograms of every still-open range (warp-aggregated atomics),
// the host picks the bin holding each target rank; ranges holding <= kCap keys are gathered
// and sorted on the host instead.  Single-key bins (e.g. the many perf == 1.0 groups, the
// upper extreme) resolve immediately.  With world > 1 the histograms are NCCL-summed and the
// gathered candidates all-gathered, so every rank selects the same value.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <vector>

#include "common.h"

namespace lscat {
namespace {

constexpr int kBins = 4096;
constexpr uint32_t kCap = 4096;
constexpr int kMaxRanges = 128;

struct Range {
  uint64_t lo, hi;   // inclusive key range
  uint32_t shift;
  uint32_t which;    // 0 perf, 1 gain
  uint32_t gather;   // 1 -> collect keys instead of a histogram
};

__device__ __forceinline__ int bin_of(const Range& r, uint64_t k) {
  if (k == r.lo) return 0;
  if (k == r.hi) return kBins - 1;
  return 1 + (int)((k - r.lo - 1) >> r.shift);
}

// kSmem: the histograms of all ranges fit in shared memory (nr <= kSmemRanges): per-CTA
// privatised counts, flushed once (hot bins such as perf == 1.0 would otherwise serialise on
// global atomics).
constexpr int kSmemRanges = 4;

template <bool kSmem>
__global__ void __launch_bounds__(256) select_pass(const double* __restrict__ perf,
                                                   const double* __restrict__ gain, uint64_t lo,
                                                   uint64_t hi, const Range* __restrict__ ranges,
                                                   int nr, uint32_t* __restrict__ hist,
                                                   uint64_t* __restrict__ cand,
                                                   uint32_t* __restrict__ cand_cnt) {
  __shared__ Range sr[kMaxRanges];
  extern __shared__ uint32_t sh_hist[];
  for (int i = threadIdx.x; i < nr; i += blockDim.x) sr[i] = ranges[i];
  if (kSmem)
    for (int i = threadIdx.x; i < nr * kBins; i += blockDim.x) sh_hist[i] = 0;
  uint32_t* H = kSmem ? sh_hist : hist;
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // A warp takes 4 chunks of 32 consecutive groups per iteration and issues all 8 loads
  // (perf, gain) before using them; whole warps iterate together (ballots, match.any).
  constexpr int kU = 4;
  const int lane = threadIdx.x & 31;
  const uint64_t wstride = stride * kU;
  for (uint64_t base = lo + (blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u)) * kU; base < hi;
       base += wstride) {
    double pv[kU], gv[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const uint64_t g = base + 32 * u + lane;
      pv[u] = g < hi ? perf[g] : __longlong_as_double(0x7FF8000000000000ll);
      gv[u] = g < hi ? gain[g] : __longlong_as_double(0x7FF8000000000000ll);
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
      for (int w = 0; w < 2; w++) {
        const double v = w ? gv[u] : pv[u];
        const bool def = !isnan(v);
        const uint64_t k = def ? (uint64_t)__double_as_longlong(v) : 0;
        for (int r = 0; r < nr; r++) {
          const Range& R = sr[r];
          if (R.which != (uint32_t)w) continue;  // warp-uniform
          const bool hit = def && k >= R.lo && k <= R.hi;
          if (!__any_sync(FULL, hit)) continue;
          if (R.gather) {
            if (hit) {
              const uint32_t idx = atomicAdd(&cand_cnt[r], 1u);
              if (idx < kCap) cand[(size_t)r * kCap + idx] = k;
            }
          } else {
            const int b = hit ? bin_of(R, k) : -1;
            // the two single-key end bins (e.g. perf == 1.0, gain == 0) are hot: count them with
            // one ballot per warp; other bins spread, one atomic per lane
            const unsigned e0 = __ballot_sync(FULL, b == 0), e1 = __ballot_sync(FULL, b == kBins - 1);
            if (lane == 0 && e0) atomicAdd(&H[(size_t)r * kBins], (uint32_t)__popc(e0));
            if (lane == 0 && e1) atomicAdd(&H[(size_t)r * kBins + kBins - 1], (uint32_t)__popc(e1));
            if (kSmem) {
              if (b > 0 && b < kBins - 1) atomicAdd(&H[(size_t)r * kBins + b], 1u);
            } else {
              const bool mid = b > 0 && b < kBins - 1;
              const unsigned peers = __match_any_sync(FULL, mid ? b : -1);
              if (mid && (__ffs(peers) - 1) == lane) atomicAdd(&H[(size_t)r * kBins + b], (uint32_t)__popc(peers));
            }
          }
        }
      }
    }
  }
  if (kSmem) {
    __syncthreads();
    for (int i = threadIdx.x; i < nr * kBins; i += blockDim.x)
      if (sh_hist[i]) atomicAdd(&hist[i], sh_hist[i]);
  }
}

struct Target {
  int which;       // 0 perf, 1 gain
  int out_index;
  uint64_t lo, hi;  // current inclusive range
  uint64_t k;       // 1-based rank inside the range
  uint64_t count;   // keys inside the range (global)
  bool done;
  uint64_t key;
};

uint32_t pick_shift(uint64_t lo, uint64_t hi) {
  if (hi - lo < 2) return 0;
  const uint64_t span = hi - lo - 2;  // max of (k - lo - 1)
  uint32_t s = 0;
  while ((span >> s) > (uint64_t)(kBins - 3)) s++;
  return s;
}


lscat_status select_percentiles(lscat_ctx* ctx, const double* pct, uint32_t npct, uint64_t n_def,
                                const uint64_t mm[4], double* out_perf, double* out_gain,
                                cudaStream_t s) {
  std::vector<Target> tg;
  for (int w = 0; w < 2; w++) {
    for (uint32_t i = 0; i < npct; i++) {
      Target t{};
      t.which = w;
      t.out_index = (int)i;
      double r = ceil(pct[i] * (double)n_def);  // nearest rank (R-13)
      t.k = r < 1.0 ? 1 : (r > (double)n_def ? n_def : (uint64_t)r);
      t.lo = mm[2 * w];
      t.hi = mm[2 * w + 1];
      t.count = n_def;
      t.done = false;
      tg.push_back(t);
    }
  }
  const ReduceState& rs = ctx->rs;
  cudaError_t err;
  Range* d_ranges = (Range*)scratch(ctx, "sel_ranges", sizeof(Range) * kMaxRanges, &err);
  if (err) return cuda_fail(ctx, err, "stats: scratch");
  uint32_t* d_hist = (uint32_t*)scratch(ctx, "sel_hist", (size_t)kMaxRanges * kBins * 4, &err);
  if (err) return cuda_fail(ctx, err, "stats: scratch");
  uint64_t* d_cand = (uint64_t*)scratch(ctx, "sel_cand", (size_t)kMaxRanges * kCap * 8, &err);
  if (err) return cuda_fail(ctx, err, "stats: scratch");
  uint32_t* d_ccnt = (uint32_t*)scratch(ctx, "sel_ccnt", kMaxRanges * 4, &err);
  if (err) return cuda_fail(ctx, err, "stats: scratch");
  uint64_t* d_gath = nullptr;
  if (ctx->world > 1) {
    d_gath = (uint64_t*)scratch(ctx, "sel_gath", (size_t)ctx->world * kMaxRanges * (kCap + 1) * 8, &err);
    if (err) return cuda_fail(ctx, err, "stats: scratch");
  }
  for (int level = 0; level < 16; level++) {
    // resolve trivially known targets
    for (auto& t : tg)
      if (!t.done && (t.lo == t.hi)) { t.done = true; t.key = t.lo; }
    // unique open ranges
    std::vector<Range> ranges;
    std::map<std::tuple<int, uint64_t, uint64_t>, int> idx;
    std::vector<int> tr(tg.size(), -1);
    for (size_t i = 0; i < tg.size(); i++) {
      Target& t = tg[i];
      if (t.done) continue;
      auto key = std::make_tuple(t.which, t.lo, t.hi);
      auto it = idx.find(key);
      if (it == idx.end()) {
        Range r{t.lo, t.hi, pick_shift(t.lo, t.hi), (uint32_t)t.which, t.count <= kCap ? 1u : 0u};
        idx[key] = (int)ranges.size();
        tr[i] = (int)ranges.size();
        ranges.push_back(r);
      } else {
        tr[i] = it->second;
      }
    }
    if (ranges.empty()) break;
    const int nr = (int)ranges.size();
    LSCAT_CUDA(ctx, cudaMemcpyAsync(d_ranges, ranges.data(), sizeof(Range) * nr, cudaMemcpyHostToDevice, s));
    LSCAT_CUDA(ctx, cudaMemsetAsync(d_hist, 0, (size_t)nr * kBins * 4, s));
    LSCAT_CUDA(ctx, cudaMemsetAsync(d_ccnt, 0, nr * 4, s));
    const uint64_t n = rs.own_hi - rs.own_lo;
    // grid: every resident CTA once (occupancy API), capped by the work (1024 groups per CTA
    // iteration)
    const uint64_t want = std::max<uint64_t>(1, (n + 1023) / 1024);
    if (n && nr <= kSmemRanges) {
      const size_t sm = (size_t)nr * kBins * 4;
      LSCAT_CUDA(ctx, cudaFuncSetAttribute(select_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      int occ = 1;
      LSCAT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, select_pass<true>, 256, sm));
      const int g2 = (int)std::min<uint64_t>(want, (uint64_t)ctx->sm_count * std::max(occ, 1));
      select_pass<true><<<g2, 256, sm, s>>>(rs.perf, rs.gain, rs.own_lo, rs.own_hi, d_ranges, nr,
                                              d_hist, d_cand, d_ccnt);
      ctx->launches++;
    } else if (n) {
      int occ = 1;
      LSCAT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, select_pass<false>, 256, 0));
      const int g2 = (int)std::min<uint64_t>(want, (uint64_t)ctx->sm_count * std::max(occ, 1));
      select_pass<false><<<g2, 256, 0, s>>>(rs.perf, rs.gain, rs.own_lo, rs.own_hi, d_ranges, nr,
                                               d_hist, d_cand, d_ccnt);
      ctx->launches++;
    }
    LSCAT_CUDA(ctx, cudaGetLastError());
    std::vector<uint32_t> hist((size_t)nr * kBins);
    std::vector<uint32_t> ccnt(nr);
    std::vector<std::vector<uint64_t>> cands(nr);
    if (ctx->world > 1) {
      lscat_status ns;
      if ((ns = ctx->comm->allreduce(ctx, {{d_hist, (size_t)nr * kBins, DT::U32, Op::Sum}}, s))) return ns;
      // candidates: [count, keys...] per range, all-gathered
      uint64_t* d_pack = (uint64_t*)scratch(ctx, "sel_pack", (size_t)kMaxRanges * (kCap + 1) * 8, &err);
      if (err) return cuda_fail(ctx, err, "stats: scratch");
      std::vector<uint32_t> lc(nr);
      LSCAT_CUDA(ctx, cudaMemcpyAsync(lc.data(), d_ccnt, nr * 4, cudaMemcpyDeviceToHost, s));
      LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
      for (int r = 0; r < nr; r++) {
        uint64_t c = std::min<uint64_t>(lc[r], kCap);
        LSCAT_CUDA(ctx, cudaMemcpyAsync(d_pack + (size_t)r * (kCap + 1), &c, 8, cudaMemcpyHostToDevice, s));
        if (c) LSCAT_CUDA(ctx, cudaMemcpyAsync(d_pack + (size_t)r * (kCap + 1) + 1, d_cand + (size_t)r * kCap, c * 8, cudaMemcpyDeviceToDevice, s));
        LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
      }
      if ((ns = ctx->comm->allgather(ctx, d_pack, d_gath, (size_t)nr * (kCap + 1), DT::U64, s))) return ns;
      std::vector<uint64_t> g((size_t)ctx->world * nr * (kCap + 1));
      LSCAT_CUDA(ctx, cudaMemcpyAsync(g.data(), d_gath, g.size() * 8, cudaMemcpyDeviceToHost, s));
      LSCAT_CUDA(ctx, cudaMemcpyAsync(hist.data(), d_hist, hist.size() * 4, cudaMemcpyDeviceToHost, s));
      LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
      for (int w = 0; w < ctx->world; w++)
        for (int r = 0; r < nr; r++) {
          const uint64_t* pk = g.data() + ((size_t)w * nr + r) * (kCap + 1);
          cands[r].insert(cands[r].end(), pk + 1, pk + 1 + pk[0]);
        }
    } else {
      // one D2H of histograms + counts, then one batch of candidate copies: <= 2 host syncs
      uint32_t* h = (uint32_t*)pinned(ctx, "sel_h", (size_t)nr * kBins * 4 + kMaxRanges * 4, &err);
      if (err) return cuda_fail(ctx, err, "stats: pinned");
      uint32_t* hc = h + (size_t)nr * kBins;
      LSCAT_CUDA(ctx, cudaMemcpyAsync(h, d_hist, (size_t)nr * kBins * 4, cudaMemcpyDeviceToHost, s));
      LSCAT_CUDA(ctx, cudaMemcpyAsync(hc, d_ccnt, nr * 4, cudaMemcpyDeviceToHost, s));
      LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
      memcpy(hist.data(), h, (size_t)nr * kBins * 4);
      size_t ncand = 0;
      for (int r = 0; r < nr; r++) ccnt[r] = ranges[r].gather ? std::min(hc[r], kCap) : 0;
      for (int r = 0; r < nr; r++) ncand += ccnt[r];
      if (ncand) {
        uint64_t* hk = (uint64_t*)pinned(ctx, "sel_k", ncand * 8, &err);
        if (err) return cuda_fail(ctx, err, "stats: pinned");
        size_t at = 0;
        for (int r = 0; r < nr; r++) {
          if (ccnt[r]) LSCAT_CUDA(ctx, cudaMemcpyAsync(hk + at, d_cand + (size_t)r * kCap, ccnt[r] * 8, cudaMemcpyDeviceToHost, s));
          at += ccnt[r];
        }
        LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
        at = 0;
        for (int r = 0; r < nr; r++) {
          cands[r].assign(hk + at, hk + at + ccnt[r]);
          at += ccnt[r];
        }
      }
    }
    for (int r = 0; r < nr; r++)
      if (ranges[r].gather) std::sort(cands[r].begin(), cands[r].end());
    for (size_t i = 0; i < tg.size(); i++) {
      Target& t = tg[i];
      if (t.done) continue;
      const int r = tr[i];
      const Range& R = ranges[r];
      if (R.gather) {
        if (cands[r].size() != t.count || t.k == 0 || t.k > t.count)
          return fail(ctx, LSCAT_ERR_STATE, "stats: percentile candidates %zu != expected %llu",
                      cands[r].size(), (unsigned long long)t.count);
        t.key = cands[r][t.k - 1];
        t.done = true;
        continue;
      }
      const uint32_t* h = hist.data() + (size_t)r * kBins;
      uint64_t cum = 0;
      int b = 0;
      for (; b < kBins; b++) {
        if (cum + h[b] >= t.k) break;
        cum += h[b];
      }
      if (b == kBins) return fail(ctx, LSCAT_ERR_STATE, "stats: percentile histogram lost keys");
      t.k -= cum;
      t.count = h[b];
      if (b == 0) { t.done = true; t.key = R.lo; continue; }
      if (b == kBins - 1) { t.done = true; t.key = R.hi; continue; }
      const uint64_t nlo = R.lo + 1 + ((uint64_t)(b - 1) << R.shift);
      uint64_t nhi = R.lo + ((uint64_t)b << R.shift);
      if (nhi > R.hi - 1) nhi = R.hi - 1;
      t.lo = nlo;
      t.hi = nhi;
    }
  }
  for (auto& t : tg) {
    if (!t.done) return fail(ctx, LSCAT_ERR_STATE, "stats: percentile selection did not converge");
    double v;
    memcpy(&v, &t.key, 8);
    (t.which ? out_gain : out_perf)[t.out_index] = v;
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
  const size_t plen = LSCAT_P_NCOUNTERS + (nb + 1) + (ng + 1) + nbb * (o->block_profile ? 3 : 1);
  std::vector<uint64_t> P(plen);
  uint64_t mm[4];
  LSCAT_CUDA(ctx, cudaMemcpyAsync(P.data(), rs.partials, plen * 8, cudaMemcpyDeviceToHost, s));
  LSCAT_CUDA(ctx, cudaMemcpyAsync(mm, rs.minmax, sizeof mm, cudaMemcpyDeviceToHost, s));
  LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  const uint64_t* C = P.data();
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
  if (o->block_profile) {  // R-22: mean of best / r_b per (matrix, block)
    const uint64_t* ps = H + nb + 1 + ng + 1 + nbb;
    const uint64_t* pc = ps + nbb;
    for (size_t i = 0; i < nbb; i++) {
      if (out->profile_count) out->profile_count[i] = pc[i];
      if (out->profile_mean) out->profile_mean[i] = pc[i] ? ((double)ps[i] * 0x1p-31) / (double)pc[i] : NAN;
    }
  }
  if (out->n_percentiles) {
    if (out->n_ratio_defined == 0) {
      for (uint32_t i = 0; i < out->n_percentiles; i++) out->pct_perf[i] = out->pct_gain[i] = NAN;
    } else {
      lscat_status st = select_percentiles(ctx, out->percentiles, out->n_percentiles,
                                           out->n_ratio_defined, mm, out->pct_perf, out->pct_gain, s);
      if (st) return st;
    }
  }
  return LSCAT_OK;
}
