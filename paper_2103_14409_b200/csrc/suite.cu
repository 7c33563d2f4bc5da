// suite.cu — a1 (register suite: buffers + on-device input generation) and a3 (one launch).
#include <cuda_bf16.h>

#include <cstring>

#include "common.h"

namespace lscat {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// uniform in [-1, 1) on a 2^-23 grid: exactly representable in fp32 (R-15)
__global__ void fill_f32(float* p, uint64_t n, uint64_t key) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = mix64(i ^ key);
    p[i] = (float)(h >> 40) * 0x1p-23f - 1.0f;
  }
}

// uniform in [-1, 1) on a 2^-7 grid: exactly representable in bf16
__global__ void fill_bf16(__nv_bfloat16* p, uint64_t n, uint64_t key) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = mix64(i ^ key);
    p[i] = __float2bfloat16_rn((float)((int)(h >> 56) - 128) * 0.0078125f);
  }
}

uint64_t buffer_key(uint64_t seed, uint32_t kernel, uint32_t n, uint32_t slot) {
  uint64_t z = seed ^ (0xA24BAED4963EE407ull * (kernel + 1)) ^ (0x9FB21C651E98DF25ull * n) ^
               (0xC13FA9A902A6328Full * (slot + 1));
  z ^= z >> 29;
  z *= 0xBF58476D1CE4E5B9ull;
  return z ^ (z >> 32);
}

void free_entry(SuiteEntry& e) {
  cudaFree(e.in0);
  cudaFree(e.in1);
  cudaFree(e.out);
  cudaFree(e.scratch);
  e = SuiteEntry{};
}

cudaError_t alloc_entry(lscat_ctx* ctx, SuiteEntry& e, cudaStream_t s) {
  const uint64_t N = e.n, N2 = N * N;
  uint64_t b0 = 0, b1 = 0, bo = 0;
  bool bf16 = false;
  switch (e.kernel) {
    case LSCAT_K_EUCLID:
    case LSCAT_K_MATVEC: b0 = 4 * N2; b1 = 4 * N; bo = 4 * N; break;
    case LSCAT_K_ROWSUM:
    case LSCAT_K_COLSUM: b0 = 4 * N2; bo = 4 * N; break;
    case LSCAT_K_TRANSPOSE:
    case LSCAT_K_STENCIL5: b0 = 4 * N2; bo = 4 * N2; break;
    case LSCAT_K_AXPY: b0 = 4 * N2; b1 = 4 * N2; bo = 4 * N2; break;
    case LSCAT_K_GEMM_BF16: b0 = 2 * N2; b1 = 2 * N2; bo = 2 * N2; bf16 = true; break;
    case LSCAT_K_SPIN: return cudaSuccess;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t err;
  if (b0 && (err = cudaMalloc(&e.in0, b0)) != cudaSuccess) return err;
  e.in0_bytes = b0;
  if (b1 && (err = cudaMalloc(&e.in1, b1)) != cudaSuccess) return err;
  e.in1_bytes = b1;
  if (bo && (err = cudaMalloc(&e.out, bo)) != cudaSuccess) return err;
  e.out_bytes = bo;
  const int grid = ctx->sm_count * 8;
  if (bf16) {
    fill_bf16<<<grid, 256, 0, s>>>((__nv_bfloat16*)e.in0, b0 / 2, buffer_key(ctx->seed, e.kernel, e.n, 0));
    fill_bf16<<<grid, 256, 0, s>>>((__nv_bfloat16*)e.in1, b1 / 2, buffer_key(ctx->seed, e.kernel, e.n, 1));
  } else {
    fill_f32<<<grid, 256, 0, s>>>((float*)e.in0, b0 / 4, buffer_key(ctx->seed, e.kernel, e.n, 0));
    if (b1) fill_f32<<<grid, 256, 0, s>>>((float*)e.in1, b1 / 4, buffer_key(ctx->seed, e.kernel, e.n, 1));
  }
  if ((err = cudaGetLastError()) != cudaSuccess) return err;
  if ((err = cudaMemsetAsync(e.out, 0, bo, s)) != cudaSuccess) return err;
  if (e.kernel == LSCAT_K_COLSUM) return colsum_prepare(e);
  if (e.kernel == LSCAT_K_GEMM_BF16) return gemm_prepare(e);
  return cudaSuccess;
}

}  // namespace
}  // namespace lscat

using namespace lscat;

extern "C" {

lscat_status lscat_register_suite(lscat_ctx* ctx, const uint32_t* kernels, uint32_t nk,
                                  const uint32_t* sizes, uint32_t ns, void* stream) {
  LSCAT_CHECK_CTX(ctx);
  if (!kernels || !sizes || nk == 0 || ns == 0)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "register_suite: empty kernel or size list");
  for (uint32_t i = 0; i < nk; i++)
    if (!kernel_table(kernels[i]))
      return fail(ctx, LSCAT_ERR_INVALID_ARG, "register_suite: unknown kernel %u", kernels[i]);
  for (uint32_t i = 0; i < ns; i++)
    if (sizes[i] == 0 || sizes[i] > 16384)
      return fail(ctx, LSCAT_ERR_INVALID_ARG, "register_suite: matrix size %u out of range", sizes[i]);
  cudaStream_t s = (cudaStream_t)stream;
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));
  LSCAT_CUDA(ctx, cudaDeviceSynchronize());
  for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
  ctx->graphs.clear();
  ctx->rot_owner = {~0u, ~0u};
  for (auto& kv : ctx->suite) free_entry(kv.second);
  ctx->suite.clear();
  for (uint32_t i = 0; i < nk; i++) {
    for (uint32_t j = 0; j < ns; j++) {
      SuiteEntry e;
      e.kernel = kernels[i];
      e.n = sizes[j];
      cudaError_t err = alloc_entry(ctx, e, s);
      if (err != cudaSuccess) {
        free_entry(e);
        return cuda_fail(ctx, err, "register_suite: allocation/initialisation");
      }
      ctx->suite[{e.kernel, e.n}] = e;
    }
  }
  LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  return LSCAT_OK;
}

lscat_status lscat_suite_buffer(lscat_ctx* ctx, uint32_t kernel, uint32_t n, uint32_t slot,
                                void** ptr, uint64_t* bytes) {
  LSCAT_CHECK_CTX(ctx);
  auto it = ctx->suite.find({kernel, n});
  if (it == ctx->suite.end() || !ptr || !bytes)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "suite_buffer: (%u, %u) not registered", kernel, n);
  const SuiteEntry& e = it->second;
  void* p = slot == 0 ? e.in0 : slot == 1 ? e.in1 : slot == 2 ? e.out : nullptr;
  uint64_t b = slot == 0 ? e.in0_bytes : slot == 1 ? e.in1_bytes : slot == 2 ? e.out_bytes : 0;
  if (!p) return fail(ctx, LSCAT_ERR_INVALID_ARG, "suite_buffer: slot %u unused", slot);
  *ptr = p;
  *bytes = b;
  return LSCAT_OK;
}

lscat_status lscat_suite_upload(lscat_ctx* ctx, uint32_t kernel, uint32_t n, uint32_t slot,
                                const void* src, uint64_t bytes, uint32_t src_mem, void* stream) {
  LSCAT_CHECK_CTX(ctx);
  void* dst = nullptr;
  uint64_t b = 0;
  if (slot > 1) return fail(ctx, LSCAT_ERR_INVALID_ARG, "suite_upload: slot %u is not an input", slot);
  lscat_status st = lscat_suite_buffer(ctx, kernel, n, slot, &dst, &b);
  if (st) return st;
  if (!src || bytes != b) return fail(ctx, LSCAT_ERR_INVALID_ARG, "suite_upload: %llu bytes, slot holds %llu",
                                      (unsigned long long)bytes, (unsigned long long)b);
  ctx->rot_owner = {~0u, ~0u};  // ROTATE copies are stale
  LSCAT_CUDA(ctx, cudaMemcpyAsync(dst, src, b, src_mem == LSCAT_MEM_HOST ? cudaMemcpyHostToDevice
                                                                        : cudaMemcpyDeviceToDevice,
                                  (cudaStream_t)stream));
  return LSCAT_OK;
}

lscat_status lscat_launch(lscat_ctx* ctx, uint32_t kernel, uint32_t n, uint32_t block,
                          void* stream) {
  LSCAT_CHECK_CTX(ctx);
  const KernelTable* t = kernel_table(kernel);
  if (!t || block < 32 || block > 1024 || block % 32)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "launch: kernel %u block %u", kernel, block);
  LaunchFn fn = t->fn[block / 32 - 1];
  if (!fn) return fail(ctx, LSCAT_ERR_UNSUPPORTED, "launch: kernel %u has no %u-thread variant", kernel, block);
  SuiteEntry spin_entry;
  const SuiteEntry* e = &spin_entry;
  if (kernel != LSCAT_K_SPIN) {
    auto it = ctx->suite.find({kernel, n});
    if (it == ctx->suite.end())
      return fail(ctx, LSCAT_ERR_STATE, "launch: (%u, %u) not registered", kernel, n);
    e = &it->second;
  }
  LaunchArgs a{e, (uint64_t)n};
  a.sms = ctx->sm_count;
  a.l2_bytes = ctx->l2_bytes;
  cudaError_t err = fn(a, (cudaStream_t)stream);
  ctx->launches++;
  if (err != cudaSuccess) return cuda_fail(ctx, err, "launch");
  return LSCAT_OK;
}

}  // extern "C"
