// selbins.h — fixed key bins of the percentile selection's sampled first level (a8, stats.cu).
//
// Keys are the IEEE bit patterns of the positive doubles (bit order == value order).  Each
// quantity has kFxBins bins in key order, fine where the paper-shaped distributions put their
// mass and single-valued at the two values that repeat (perf == 1 <=> gain == 0 <=> t == b):
//   perf in (0, 1]:  [0] perf < 1/4, [1 .. 2048] 1/4 <= perf < 1 in 1024 bins per binade
//                    (key >> 42), [2049] perf == 1, [2050] unused;
//   gain in [0, ..): [0] gain == 0, [1] 0 < gain < 2^-13, [2 .. 2049] 2^-13 <= gain < 8 in 128
//                    bins per binade (key >> 45), [2050] gain >= 8.
#pragma once
#include <cstdint>

namespace lscat {

constexpr uint32_t kFxBins = 2051;
constexpr uint64_t kPerfLo = 0x3FD0000000000000ull;  // 0.25
constexpr uint64_t kPerfOne = 0x3FF0000000000000ull; // 1.0
constexpr int kPerfShift = 42;
constexpr uint64_t kGainLo = 0x3F20000000000000ull;  // 2^-13
constexpr uint64_t kGainHi = 0x4020000000000000ull;  // 8.0
constexpr int kGainShift = 45;

// bin of a perf key (0 < perf <= 1) and of a gain key (gain >= 0)
__host__ __device__ __forceinline__ uint32_t fx_perf_bin(uint64_t k) {
  if (k >= kPerfOne) return kFxBins - 2;
  return k < kPerfLo ? 0u : 1u + (uint32_t)((k >> kPerfShift) - (kPerfLo >> kPerfShift));
}
__host__ __device__ __forceinline__ uint32_t fx_gain_bin(uint64_t k) {
  if (k == 0) return 0u;
  return k < kGainLo ? 1u : (k >= kGainHi ? kFxBins - 1 : 2u + (uint32_t)((k >> kGainShift) - (kGainLo >> kGainShift)));
}
// the same bins from the key's high 32 bits (every bin edge lies on a multiple of 2^42): the
// selection pass bins in 32-bit arithmetic.  Valid only for keys of the counted bins.
__host__ __device__ __forceinline__ uint32_t fx_perf_bin_hi(uint32_t h) {
  return h < (uint32_t)(kPerfLo >> 32) ? 0u : 1u + ((h >> (kPerfShift - 32)) - (uint32_t)(kPerfLo >> kPerfShift));
}
__host__ __device__ __forceinline__ uint32_t fx_gain_bin_hi(uint32_t h) {
  return h < (uint32_t)(kGainLo >> 32) ? 1u
         : (h >= (uint32_t)(kGainHi >> 32) ? kFxBins - 1 : 2u + ((h >> (kGainShift - 32)) - (uint32_t)(kGainLo >> kGainShift)));
}

// inclusive key range of bin b of quantity w (0 perf, 1 gain), before clipping to [min, max]
__host__ __device__ __forceinline__ void fx_bin_range(uint32_t w, uint32_t b, uint64_t* lo, uint64_t* hi) {
  if (w == 0) {
    if (b == 0) { *lo = 0; *hi = kPerfLo - 1; }
    else if (b >= kFxBins - 2) { *lo = *hi = kPerfOne; }
    else { *lo = kPerfLo + ((uint64_t)(b - 1) << kPerfShift); *hi = *lo + ((1ull << kPerfShift) - 1); }
  } else {
    if (b == 0) { *lo = *hi = 0; }
    else if (b == 1) { *lo = 1; *hi = kGainLo - 1; }
    else if (b == kFxBins - 1) { *lo = kGainHi; *hi = ~0ull; }
    else { *lo = kGainLo + ((uint64_t)(b - 2) << kGainShift); *hi = *lo + ((1ull << kGainShift) - 1); }
  }
}

}  // namespace lscat
