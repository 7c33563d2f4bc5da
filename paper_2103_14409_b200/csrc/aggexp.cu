// aggexp.cu — the paper's timing-aggregation experiment:
// "Five different simple methods were tested out, by creating a dataset of 100 000 run times,
// then randomly selecting ten and aggregating, by repeating this process the variations after
// aggregation can be measured.  Out of the different aggregation methods tested the median
// performed the best".  Readings (R-23): the five methods are mean, median, min,
// max and the 20 % trimmed mean (drop floor(k/10) lowest and highest); k values are drawn
// without replacement by Floyd's algorithm from a counter-based generator; the variation of a
// method = population standard deviation of its `reps` aggregates / their mean.
//
// One thread per repetition: draw, insertion-sort k <= 64 values, five aggregates (double,
// sums in ascending order); then one CTA reduces each method's aggregates in a fixed order.
#include <cmath>

#include "common.h"

namespace lscat {
namespace {

constexpr int kMaxK = 64;

__device__ __forceinline__ uint64_t smix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// uniform integer in [0, m] for repetition `rep`, draw `j` (multiply-shift on 32 random bits)
__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t rep, uint64_t j, uint64_t m) {
  const uint64_t h = smix(smix(seed ^ (rep * 0xD1B54A32D192ED03ull)) ^ j);
  return ((h >> 32) * (m + 1)) >> 32;
}

__global__ void aggexp_reps(const float* __restrict__ pool, uint64_t n, uint32_t k, uint32_t reps,
                            uint64_t seed, double* __restrict__ agg /* [5][reps] */) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= reps) return;
  uint64_t idx[kMaxK];
  // Floyd: for j = n-k .. n-1 pick t in [0, j]; take t unless already taken, else j
  for (uint32_t i = 0; i < k; i++) {
    const uint64_t j = n - k + i;
    const uint64_t t = draw(seed, r, j, j);
    bool taken = false;
    for (uint32_t q = 0; q < i; q++) taken |= (idx[q] == t);
    idx[i] = taken ? j : t;
  }
  float v[kMaxK];
  for (uint32_t i = 0; i < k; i++) v[i] = pool[idx[i]];
  for (uint32_t i = 1; i < k; i++) {  // insertion sort, ascending
    const float x = v[i];
    int q = (int)i - 1;
    while (q >= 0 && v[q] > x) { v[q + 1] = v[q]; q--; }
    v[q + 1] = x;
  }
  double s = 0.0;
  for (uint32_t i = 0; i < k; i++) s = __dadd_rn(s, (double)v[i]);
  const double mean = __ddiv_rn(s, (double)k);
  const double med = (k & 1) ? (double)v[k / 2] : __dmul_rn(__dadd_rn((double)v[k / 2 - 1], (double)v[k / 2]), 0.5);
  const uint32_t cut = k / 10;
  double st = 0.0;
  for (uint32_t i = cut; i < k - cut; i++) st = __dadd_rn(st, (double)v[i]);
  const double trim = __ddiv_rn(st, (double)(k - 2 * cut));
  agg[0 * (size_t)reps + r] = mean;
  agg[1 * (size_t)reps + r] = med;
  agg[2 * (size_t)reps + r] = (double)v[0];
  agg[3 * (size_t)reps + r] = (double)v[k - 1];
  agg[4 * (size_t)reps + r] = trim;
}

// one CTA of 256 threads per method: mean, then population variance, fixed-order tree
__global__ void aggexp_spread(const double* __restrict__ agg, uint32_t reps, double* __restrict__ out) {
  __shared__ double red[256];
  const double* a = agg + (size_t)blockIdx.x * reps;
  double s = 0.0;
  for (uint32_t i = threadIdx.x; i < reps; i += 256) s = __dadd_rn(s, a[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  const double mean = __ddiv_rn(red[0], (double)reps);
  __syncthreads();
  double q = 0.0;
  for (uint32_t i = threadIdx.x; i < reps; i += 256) {
    const double d = __dsub_rn(a[i], mean);
    q = __dadd_rn(q, __dmul_rn(d, d));
  }
  red[threadIdx.x] = q;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = mean;
    out[2 * blockIdx.x + 1] = __ddiv_rn(sqrt(__ddiv_rn(red[0], (double)reps)), mean);
  }
}

}  // namespace
}  // namespace lscat

using namespace lscat;

extern "C" lscat_status lscat_aggregation_experiment(lscat_ctx* ctx, const float* pool, uint64_t n_pool,
                                                     uint32_t k, uint32_t reps, uint64_t seed,
                                                     double* spread, double* mean_of_aggregates,
                                                     double* aggregates, void* stream) {
  LSCAT_CHECK_CTX(ctx);
  if (!pool || !spread || k == 0 || k > kMaxK || reps == 0 || n_pool < k)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "aggregation_experiment: need 1 <= k <= %d <= n_pool, reps >= 1", kMaxK);
  cudaStream_t s = (cudaStream_t)stream;
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));
  cudaError_t err;
  double* agg = aggregates;
  if (!agg) {
    agg = (double*)scratch(ctx, "aggexp", (size_t)5 * reps * 8, &err);
    if (err) return cuda_fail(ctx, err, "aggregation_experiment: scratch");
  }
  double* res = (double*)scratch(ctx, "aggexp_out", 10 * 8, &err);
  if (err) return cuda_fail(ctx, err, "aggregation_experiment: scratch");
  aggexp_reps<<<(reps + 127) / 128, 128, 0, s>>>(pool, n_pool, k, reps, seed, agg);
  aggexp_spread<<<5, 256, 0, s>>>(agg, reps, res);
  ctx->launches += 2;
  LSCAT_CUDA(ctx, cudaGetLastError());
  double h[10];
  LSCAT_CUDA(ctx, cudaMemcpyAsync(h, res, sizeof h, cudaMemcpyDeviceToHost, s));
  LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  for (int i = 0; i < 5; i++) {
    spread[i] = h[2 * i + 1];
    if (mean_of_aggregates) mean_of_aggregates[i] = h[2 * i];
  }
  return LSCAT_OK;
}
