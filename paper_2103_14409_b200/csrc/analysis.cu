// analysis.cu — the paper's two side analyses adjacent to the sweep:
//   * occupancy-API block: the block size CUDA's occupancy calculator
//     picks for a kernel — cudaOccupancyMaxPotentialBlockSizeVariableSMem and
//     cudaOccupancyMaxActiveBlocksPerMultiprocessor on every candidate's compiled function,
//     the most resident warps per SM winning, ties to the larger block (the API's rule).  It depends on the kernel's
//     resources only, never on the matrix size ("insensitive to matrix sizes").  Its
//     quality is then measured with lscat_reduce_table by setting largest_block_id to it.
//   * timeout economics: how many sweep points finish within a timeout tau, from the
//     runtime table: a point's time is (W + K R) x its per-launch runtime.
#include <algorithm>
#include <cmath>

#include "common.h"

namespace lscat {
namespace {

constexpr int kMaxTaus = 64;

// counts[i] = #rows with a result whose point time (W + K R) * runtime_ms * 1e-3 <= taus[i]
__global__ void timeout_curve_kernel(const float* __restrict__ rt, uint64_t n, double launches,
                                     const double* __restrict__ taus, int nt,
                                     unsigned long long* __restrict__ counts) {
  __shared__ double st[kMaxTaus];
  __shared__ unsigned int sc[kMaxTaus];
  for (int i = threadIdx.x; i < nt; i += blockDim.x) { st[i] = taus[i]; sc[i] = 0; }
  __syncthreads();
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const float v = rt[r];
    const uint32_t b = __float_as_uint(v);
    if (b - 1u >= 0x7F7FFFFFu) continue;  // no result (NaN, inf, <= 0)
    const double t = __dmul_rn(__dmul_rn(launches, (double)v), 1e-3);
    for (int i = 0; i < nt; i++)
      if (t <= st[i]) atomicAdd(&sc[i], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nt; i += blockDim.x)
    if (sc[i]) atomicAdd(&counts[i], (unsigned long long)sc[i]);
}

}  // namespace
}  // namespace lscat

using namespace lscat;

extern "C" {

lscat_status lscat_occupancy_block(lscat_ctx* ctx, uint32_t kernel, const uint16_t* blocks,
                                   uint32_t n_blocks, uint32_t* out_block_id, lscat_occupancy_info* info) {
  LSCAT_CHECK_CTX(ctx);
  const KernelTable* t = kernel_table(kernel);
  if (!t || !out_block_id || !block_list_ok(blocks, n_blocks))
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "occupancy_block: bad kernel or block list");
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));
  int best = -1, best_w = -1;
  for (uint32_t i = 0; i < n_blocks; i++) {
    const int B = blocks[i];
    lscat_occupancy_info in{};
    in.threads = (uint32_t)B;
    AttrFn af = t->attrs[B / 32 - 1];
    const void* f = nullptr;
    size_t dyn = 0;
    if (af && af(&f, &dyn) == cudaSuccess && f) {
      cudaFuncAttributes fa{};
      LSCAT_CUDA(ctx, cudaFuncGetAttributes(&fa, f));
      in.regs_per_thread = fa.numRegs;
      in.static_smem = (int32_t)fa.sharedSizeBytes;
      in.dynamic_smem = (int32_t)dyn;
      in.max_threads_per_block = fa.maxThreadsPerBlock;
      int nb = 0;
      LSCAT_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, B, dyn));
      in.blocks_per_sm = nb;
      in.warps_per_sm = nb * B / 32;
      int min_grid = 0, blk = 0;
      LSCAT_CUDA(ctx, cudaOccupancyMaxPotentialBlockSizeVariableSMem(
                          &min_grid, &blk, f, [dyn](int) { return dyn; }, B));
      in.api_block = blk;
      in.api_min_grid = min_grid;
    }
    cudaGetLastError();
    if (info) info[i] = in;
    if (in.warps_per_sm > 0 && in.warps_per_sm >= best_w) { best_w = in.warps_per_sm; best = (int)i; }  // ties -> larger
  }
  if (best < 0) return fail(ctx, LSCAT_ERR_UNSUPPORTED, "occupancy_block: no block size is launchable");
  *out_block_id = (uint32_t)best;
  return LSCAT_OK;
}

lscat_status lscat_timeout_curve(lscat_ctx* ctx, const lscat_table* T, uint32_t warmup, uint32_t brackets,
                                 uint32_t launches_per_bracket, const double* taus, uint32_t n_taus,
                                 uint64_t* counts, void* stream) {
  LSCAT_CHECK_CTX(ctx);
  if (!T || !T->runtime_ms || T->mem != LSCAT_MEM_DEVICE || !taus || !counts || n_taus == 0 ||
      n_taus > (uint32_t)kMaxTaus)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "timeout_curve: device table, 1..%d host taus and counts", kMaxTaus);
  cudaStream_t s = (cudaStream_t)stream;
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));
  cudaError_t err;
  double* d_t = (double*)scratch(ctx, "tc_taus", n_taus * 8, &err);
  if (err) return cuda_fail(ctx, err, "timeout_curve: scratch");
  unsigned long long* d_c = (unsigned long long*)scratch(ctx, "tc_counts", n_taus * 8, &err);
  if (err) return cuda_fail(ctx, err, "timeout_curve: scratch");
  LSCAT_CUDA(ctx, cudaMemcpyAsync(d_t, taus, n_taus * 8, cudaMemcpyHostToDevice, s));
  LSCAT_CUDA(ctx, cudaMemsetAsync(d_c, 0, n_taus * 8, s));
  const double launches = (double)warmup + (double)brackets * (double)launches_per_bracket;
  if (T->n_rows) {
    const int grid = (int)std::min<uint64_t>((uint64_t)ctx->sm_count * 4, (T->n_rows + 255) / 256);
    timeout_curve_kernel<<<grid, 256, 0, s>>>(T->runtime_ms, T->n_rows, launches, d_t, (int)n_taus, d_c);
    ctx->launches++;
    LSCAT_CUDA(ctx, cudaGetLastError());
  }
  LSCAT_CUDA(ctx, cudaMemcpyAsync(counts, d_c, n_taus * 8, cudaMemcpyDeviceToHost, s));
  LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  return LSCAT_OK;
}

}  // extern "C"
