// ingest.cu — SURVEY §8(f) #3: turn an unordered runtime dataframe (the paper's Pandas rows of
// parameter combination, path, function name and result) into a grouped runtime table:
// groups = distinct (kernel, matrix) in ascending order, rows inside a group ascending by block
// id, CSR offsets.  Stable LSD radix sort of a compressed key (kernel, matrix, block) ->
// (kernel * M + matrix) * L + block with 8-bit digits, only as many passes as the key needs
// (19 683 kernels x 8 matrices x 32 blocks: 23 bits, 3 passes):
//   hist:    per-CTA digit counts of a 4096-element tile (shared-memory atomics)
//   scan:    one CTA, exclusive scan of the [digit][tile] counts (digit-major = stable order)
//   scatter: each warp owns 512 consecutive elements (16 coalesced chunks of 32 in registers);
//            per-warp digit counts, an exclusive prefix over the CTA's warps, then in chunk order
//            rank = tile offset + warp prefix + running count + rank among equal lanes
//            (match.any): a stable counting sort per pass.
// Then gather the payload, flag group starts, scan the flags (3-phase) and emit offsets.
#include <algorithm>

#include "common.h"

namespace lscat {
namespace {

constexpr int kTPB = 256, kItems = 16, kTile = kTPB * kItems, kWarpsPB = kTPB / 32;

__global__ void make_keys(const uint32_t* __restrict__ kern, const uint32_t* __restrict__ mat,
                          const uint16_t* __restrict__ blk, uint64_t n, uint64_t M, uint64_t L,
                          uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    keys[i] = ((uint64_t)kern[i] * M + mat[i]) * L + blk[i];
    idx[i] = (uint32_t)i;
  }
}

__global__ void max3(const uint32_t* __restrict__ kern, const uint32_t* __restrict__ mat,
                     const uint16_t* __restrict__ blk, uint64_t n, unsigned int* __restrict__ out) {
  uint32_t a = 0, b = 0, c = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    a = max(a, kern[i]);
    b = max(b, mat[i]);
    c = max(c, (uint32_t)blk[i]);
  }
  a = __reduce_max_sync(0xffffffffu, a);
  b = __reduce_max_sync(0xffffffffu, b);
  c = __reduce_max_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) { atomicMax(&out[0], a); atomicMax(&out[1], b); atomicMax(&out[2], c); }
}

__global__ void __launch_bounds__(kTPB) radix_hist(const uint64_t* __restrict__ keys, uint64_t n, int shift,
                                                   uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  for (int i = threadIdx.x; i < kTile; i += kTPB) {
    const uint64_t j = base + i;
    if (j < n) atomicAdd(&cnt[(keys[j] >> shift) & 255], 1u);
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = cnt[threadIdx.x];
}

// exclusive scan in place of m u32 values, one CTA of 1024 threads (chunked)
__global__ void __launch_bounds__(1024) scan_single(uint32_t* __restrict__ v, uint64_t m, uint32_t* __restrict__ total) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t b = 0; b < m; b += 1024) {
    const uint64_t i = b + threadIdx.x;
    const uint32_t x = i < m ? v[i] : 0u;
    uint32_t s = x;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if ((threadIdx.x & 31) >= o) s += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t w = ws[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      ws[threadIdx.x] = w;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t wpre = (threadIdx.x >> 5) ? ws[(threadIdx.x >> 5) - 1] : 0u;
    if (i < m) v[i] = carry + wpre + s - x;
    __syncthreads();
    if (threadIdx.x == 0) carry += ws[31];
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kTPB) radix_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                      uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                      uint64_t n, int shift, const uint32_t* __restrict__ offs) {
  __shared__ uint32_t wc[kWarpsPB][256];
  __shared__ uint32_t toff[256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarpsPB * 256; i += kTPB) (&wc[0][0])[i] = 0;
  toff[threadIdx.x] = offs[(size_t)threadIdx.x * gridDim.x + blockIdx.x];
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kTile + (uint64_t)w * (kItems * 32);
  uint64_t k[kItems];
  uint32_t v[kItems];
#pragma unroll
  for (int c = 0; c < kItems; c++) {
    const uint64_t j = base + c * 32 + lane;
    k[c] = j < n ? kin[j] : ~0ull;
    v[c] = j < n ? vin[j] : 0u;
  }
  const unsigned lt = (1u << lane) - 1u;
  // per-warp digit histogram
#pragma unroll
  for (int c = 0; c < kItems; c++) {
    const uint64_t j = base + c * 32 + lane;
    const int d = j < n ? (int)((k[c] >> shift) & 255) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d >= 0 && (__ffs(peers) - 1) == lane) wc[w][d] += __popc(peers);
    __syncwarp();  // the next chunk's leader for d may be another lane
  }
  __syncthreads();
  {  // exclusive prefix over the CTA's warps, per digit
    const int d = threadIdx.x;
    uint32_t run = 0;
    for (int q = 0; q < kWarpsPB; q++) {
      const uint32_t t = wc[q][d];
      wc[q][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < kItems; c++) {
    const uint64_t j = base + c * 32 + lane;
    const int d = j < n ? (int)((k[c] >> shift) & 255) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    uint32_t pos = 0;
    if (d >= 0) pos = toff[d] + wc[w][d] + __popc(peers & lt);
    __syncwarp();
    if (d >= 0 && (__ffs(peers) - 1) == lane) wc[w][d] += __popc(peers);
    __syncwarp();
    if (d >= 0) {
      kout[pos] = k[c];
      vout[pos] = v[c];
    }
    __syncwarp();
  }
}

// gather the payload in sorted order; flag group starts (key / L changes) and duplicates
__global__ void gather_flag(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx, uint64_t n, uint64_t L,
                            const float* __restrict__ rt, const uint16_t* __restrict__ blk, const uint8_t* __restrict__ st,
                            float* __restrict__ rt_out, uint16_t* __restrict__ blk_out, uint8_t* __restrict__ st_out,
                            uint32_t* __restrict__ flag, unsigned long long* __restrict__ dups) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = idx[i];
    rt_out[i] = rt[s];
    blk_out[i] = blk[s];
    if (st_out) st_out[i] = st ? st[s] : (uint8_t)0;
    const bool start = i == 0 || keys[i] / L != keys[i - 1] / L;
    flag[i] = start;
    if (i > 0 && keys[i] == keys[i - 1]) atomicAdd(dups, 1ull);
  }
}

// 3-phase exclusive scan of u32 flags: per-block sums, scan of the sums, add back
__global__ void __launch_bounds__(1024) block_sums(const uint32_t* __restrict__ f, uint64_t n, uint32_t* __restrict__ sums) {
  __shared__ uint32_t s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  const uint64_t i = blockIdx.x * 1024ull + threadIdx.x;
  const uint32_t x = i < n ? f[i] : 0u;
  const uint32_t w = __reduce_add_sync(0xffffffffu, x);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(&s, w);
  __syncthreads();
  if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) emit_groups(const uint32_t* __restrict__ f, const uint64_t* __restrict__ keys,
                                                    uint64_t n, uint64_t M, uint64_t L,
                                                    const uint32_t* __restrict__ sums_scanned,
                                                    int64_t* __restrict__ off, uint32_t* __restrict__ gk,
                                                    uint32_t* __restrict__ gm) {
  __shared__ uint32_t ws[32];
  const uint64_t i = blockIdx.x * 1024ull + threadIdx.x;
  const uint32_t x = i < n ? f[i] : 0u;
  uint32_t s = x;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) >= o) s += y;
  }
  if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t w = ws[threadIdx.x];
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (threadIdx.x >= o) w += y;
    }
    ws[threadIdx.x] = w;
  }
  __syncthreads();
  const uint32_t g = sums_scanned[blockIdx.x] + ((threadIdx.x >> 5) ? ws[(threadIdx.x >> 5) - 1] : 0u) + s - x;
  if (i < n && x) {
    const uint64_t km = keys[i] / L;
    off[g] = (int64_t)i;
    if (gk) gk[g] = (uint32_t)(km / M);
    if (gm) gm[g] = (uint32_t)(km % M);
  }
}

}  // namespace
}  // namespace lscat

using namespace lscat;

extern "C" lscat_status lscat_ingest(lscat_ctx* ctx, const uint32_t* kernel, const uint32_t* matrix,
                                     const uint16_t* block_id, const float* runtime, const uint8_t* status,
                                     uint64_t n, lscat_table* out, uint64_t* n_duplicates, void* stream) {
  LSCAT_CHECK_CTX(ctx);
  if (!out || out->mem != LSCAT_MEM_DEVICE || !out->runtime_ms || !out->block_id || !out->group_offset ||
      (n && (!kernel || !matrix || !block_id || !runtime)) || out->cap_rows < n || n >= (1ull << 32))
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "ingest: device inputs, a device table with cap_rows >= n < 2^32");
  cudaStream_t s = (cudaStream_t)stream;
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));
  cudaError_t err;
  if (n == 0) {
    LSCAT_CUDA(ctx, cudaMemsetAsync(out->group_offset, 0, 8, s));
    LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
    out->n_rows = out->n_groups = 0;
    out->rows_per_group = 0;
    out->first_group = 0;
    if (n_duplicates) *n_duplicates = 0;
    return LSCAT_OK;
  }
  unsigned int* d_max = (unsigned int*)scratch(ctx, "ing_max", 16, &err);
  if (err) return cuda_fail(ctx, err, "ingest: scratch");
  LSCAT_CUDA(ctx, cudaMemsetAsync(d_max, 0, 16, s));
  const int g1 = (int)std::min<uint64_t>((uint64_t)ctx->sm_count * 8, (n + 255) / 256);
  max3<<<g1, 256, 0, s>>>(kernel, matrix, block_id, n, d_max);
  unsigned int hmax[3];
  LSCAT_CUDA(ctx, cudaMemcpyAsync(hmax, d_max, 12, cudaMemcpyDeviceToHost, s));
  LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  const uint64_t M = (uint64_t)hmax[1] + 1, L = (uint64_t)hmax[2] + 1;
  const uint64_t kmax = ((uint64_t)hmax[0] * M + hmax[1]) * L + hmax[2];
  int bits = 0;
  while (bits < 64 && (kmax >> bits)) bits++;
  const int passes = std::max(1, (bits + 7) / 8);
  uint64_t* k0 = (uint64_t*)scratch(ctx, "ing_k0", n * 8, &err);
  if (err) return cuda_fail(ctx, err, "ingest: scratch");
  uint64_t* k1 = (uint64_t*)scratch(ctx, "ing_k1", n * 8, &err);
  if (err) return cuda_fail(ctx, err, "ingest: scratch");
  uint32_t* v0 = (uint32_t*)scratch(ctx, "ing_v0", n * 4, &err);
  if (err) return cuda_fail(ctx, err, "ingest: scratch");
  uint32_t* v1 = (uint32_t*)scratch(ctx, "ing_v1", n * 4, &err);
  if (err) return cuda_fail(ctx, err, "ingest: scratch");
  const uint64_t tiles = (n + kTile - 1) / kTile;
  uint32_t* hist = (uint32_t*)scratch(ctx, "ing_hist", tiles * 256 * 4, &err);
  if (err) return cuda_fail(ctx, err, "ingest: scratch");
  make_keys<<<g1, 256, 0, s>>>(kernel, matrix, block_id, n, M, L, k0, v0);
  ctx->launches += 2;
  for (int p = 0; p < passes; p++) {
    radix_hist<<<(unsigned)tiles, kTPB, 0, s>>>(k0, n, 8 * p, hist);
    scan_single<<<1, 1024, 0, s>>>(hist, tiles * 256, nullptr);
    radix_scatter<<<(unsigned)tiles, kTPB, 0, s>>>(k0, v0, k1, v1, n, 8 * p, hist);
    ctx->launches += 3;
    std::swap(k0, k1);
    std::swap(v0, v1);
  }
  uint32_t* flag = (uint32_t*)scratch(ctx, "ing_flag", n * 4, &err);
  if (err) return cuda_fail(ctx, err, "ingest: scratch");
  unsigned long long* d_dup = (unsigned long long*)scratch(ctx, "ing_dup", 16, &err);
  if (err) return cuda_fail(ctx, err, "ingest: scratch");
  LSCAT_CUDA(ctx, cudaMemsetAsync(d_dup, 0, 16, s));
  gather_flag<<<g1, 256, 0, s>>>(k0, v0, n, L, runtime, block_id, status, out->runtime_ms, out->block_id,
                                 out->status, flag, d_dup);
  const uint64_t nb = (n + 1023) / 1024;
  uint32_t* sums = (uint32_t*)scratch(ctx, "ing_sums", (nb + 1) * 4, &err);
  if (err) return cuda_fail(ctx, err, "ingest: scratch");
  block_sums<<<(unsigned)nb, 1024, 0, s>>>(flag, n, sums);
  scan_single<<<1, 1024, 0, s>>>(sums, nb, sums + nb);
  uint32_t hG = 0;
  unsigned long long hdup = 0;
  LSCAT_CUDA(ctx, cudaMemcpyAsync(&hG, sums + nb, 4, cudaMemcpyDeviceToHost, s));
  LSCAT_CUDA(ctx, cudaMemcpyAsync(&hdup, d_dup, 8, cudaMemcpyDeviceToHost, s));
  LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  if (out->cap_groups < hG)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "ingest: %u groups > cap_groups %llu", hG,
                (unsigned long long)out->cap_groups);
  emit_groups<<<(unsigned)nb, 1024, 0, s>>>(flag, k0, n, M, L, sums, out->group_offset, out->group_kernel,
                                            out->group_matrix);
  ctx->launches += 4;
  const int64_t nn = (int64_t)n;
  LSCAT_CUDA(ctx, cudaMemcpyAsync(out->group_offset + hG, &nn, 8, cudaMemcpyHostToDevice, s));
  LSCAT_CUDA(ctx, cudaGetLastError());
  LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  out->n_rows = n;
  out->n_groups = hG;
  out->rows_per_group = 0;
  out->first_group = 0;
  if (n_duplicates) *n_duplicates = hdup;
  if (hdup) return fail(ctx, LSCAT_ERR_INVALID_ARG, "ingest: %llu duplicated (kernel, matrix, block) rows", hdup);
  return LSCAT_OK;
}
