// ctx.cu — context, errors, scratch, NCCL communicator, work model and the sweep planner (a2).
#include <algorithm>
#include <cstdarg>
#include <cstring>
#include <numeric>
#include <queue>

#include <mutex>

#include "common.h"

namespace lscat {

lscat_status fail(lscat_ctx* ctx, lscat_status s, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return s;
}

bool is_sticky(cudaError_t e) {
  switch (e) {
    case cudaErrorIllegalAddress:
    case cudaErrorLaunchFailure:
    case cudaErrorIllegalInstruction:
    case cudaErrorMisalignedAddress:
    case cudaErrorInvalidAddressSpace:
    case cudaErrorInvalidPc:
    case cudaErrorHardwareStackError:
    case cudaErrorAssert:
    case cudaErrorECCUncorrectable:
    case cudaErrorLaunchTimeout:
      return true;
    default:
      return false;
  }
}

lscat_status cuda_fail(lscat_ctx* ctx, cudaError_t e, const char* what) {
  if (ctx) {
    ctx->err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    if (is_sticky(e)) ctx->poisoned = true;
  }
  if (e == cudaErrorMemoryAllocation) return LSCAT_ERR_OOM;
  return LSCAT_ERR_CUDA;
}

void* scratch(lscat_ctx* ctx, const char* name, size_t bytes, cudaError_t* err) {
  *err = cudaSuccess;
  DevBuf& b = ctx->scratch[name];
  if (b.bytes < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    size_t want = std::max(bytes, (size_t)256);
    *err = cudaMalloc(&b.p, want);
    ctx->scratch_gen++;
    if (*err != cudaSuccess) return nullptr;
    b.bytes = want;
  }
  return b.p;
}

void* pinned(lscat_ctx* ctx, const char* name, size_t bytes, cudaError_t* err) {
  *err = cudaSuccess;
  DevBuf& b = ctx->pinned[name];
  if (b.bytes < bytes) {
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.bytes = 0;
    size_t want = std::max(bytes, (size_t)4096);
    *err = cudaMallocHost(&b.p, want);
    ctx->scratch_gen++;
    if (*err != cudaSuccess) return nullptr;
    b.bytes = want;
  }
  return b.p;
}

// Algorithmic HBM bytes and FLOPs of one launch.
void kernel_work(uint32_t k, uint32_t n, uint64_t* bytes, uint64_t* flops) {
  const uint64_t N = n, N2 = N * N;
  uint64_t b = 0, f = 0;
  switch (k) {
    case LSCAT_K_EUCLID: b = 4 * N2 + 8 * N; f = 3 * N2; break;   // read A, q; write d
    case LSCAT_K_MATVEC: b = 4 * N2 + 8 * N; f = 2 * N2; break;   // read A, x; write y
    case LSCAT_K_ROWSUM: b = 4 * N2 + 4 * N; f = N2; break;       // read A; write r
    case LSCAT_K_COLSUM: b = 4 * N2 + 4 * N; f = N2; break;       // read A; write c
    case LSCAT_K_TRANSPOSE: b = 8 * N2; f = 0; break;             // read A; write B
    case LSCAT_K_AXPY: b = 12 * N2; f = 2 * N2; break;            // read x, y; write z
    case LSCAT_K_STENCIL5: b = 8 * N2; f = 6 * N2; break;         // read A; write out
    case LSCAT_K_GEMM_BF16: b = 6 * N2; f = 2 * N2 * N; break;    // A, Bt, C in bf16
    default: break;
  }
  *bytes = b;
  *flops = f;
}

bool block_list_ok(const uint16_t* blocks, uint32_t n) {
  if (!blocks || n == 0 || n > (uint32_t)kMaxBlockIdx) return false;
  for (uint32_t i = 0; i < n; i++) {
    if (blocks[i] < 32 || blocks[i] > 1024 || blocks[i] % 32) return false;
    if (i && blocks[i] <= blocks[i - 1]) return false;  // unique, ascending -> ids
  }
  return true;
}

const KernelTable* kernel_table(uint32_t kernel) {
  switch (kernel) {
    case LSCAT_K_EUCLID: return &table_euclid();
    case LSCAT_K_MATVEC: return &table_matvec();
    case LSCAT_K_ROWSUM: return &table_rowsum();
    case LSCAT_K_COLSUM: return &table_colsum();
    case LSCAT_K_TRANSPOSE: return &table_transpose();
    case LSCAT_K_AXPY: return &table_axpy();
    case LSCAT_K_STENCIL5: return &table_stencil5();
    case LSCAT_K_GEMM_BF16: return &table_gemm();
    case LSCAT_K_SPIN: return &table_spin();
    default: return nullptr;
  }
}

}  // namespace lscat

using namespace lscat;

namespace lscat {
cudaError_t ensure_smem_attr(const void* func, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static std::mutex m;
  static std::map<std::pair<const void*, int>, size_t> set;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(m);
  size_t& cur = set[{func, dev}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}
}  // namespace lscat

extern "C" {

int lscat_abi_version(void) { return LSCAT_ABI_VERSION; }

const char* lscat_status_string(lscat_status s) {
  switch (s) {
    case LSCAT_OK: return "ok";
    case LSCAT_ERR_INVALID_ARG: return "invalid argument";
    case LSCAT_ERR_CUDA: return "cuda error";
    case LSCAT_ERR_OOM: return "out of memory";
    case LSCAT_ERR_NCCL: return "nccl error";
    case LSCAT_ERR_STATE: return "bad state";
    case LSCAT_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown";
}

lscat_status lscat_ctx_create(int device, uint64_t seed, lscat_ctx** out) {
  if (!out) return LSCAT_ERR_INVALID_ARG;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return LSCAT_ERR_CUDA;  // no CPU fallback
  if (device < 0 || device >= ndev) return LSCAT_ERR_INVALID_ARG;
  if ((e = cudaSetDevice(device)) != cudaSuccess) return LSCAT_ERR_CUDA;
  auto* c = new lscat_ctx();
  c->device = device;
  c->seed = seed;
  int l2 = 0;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
  c->l2_bytes = (size_t)l2;
  if (cudaStreamCreateWithFlags(&c->capture_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return LSCAT_ERR_CUDA;
  }
  *out = c;
  return LSCAT_OK;
}

void lscat_ctx_destroy(lscat_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : c->sel_graphs) cudaGraphExecDestroy(kv.second);
  for (auto& rg : c->red_graphs)
    if (rg.gx) cudaGraphExecDestroy(rg.gx);
  for (auto ev : c->events) cudaEventDestroy(ev);
  for (auto& kv : c->suite) {
    cudaFree(kv.second.in0);
    cudaFree(kv.second.in1);
    cudaFree(kv.second.out);
    cudaFree(kv.second.scratch);
  }
  for (auto& kv : c->scratch) cudaFree(kv.second.p);
  for (auto& kv : c->pinned) cudaFreeHost(kv.second.p);
  delete c->comm;
  if (c->capture_stream) cudaStreamDestroy(c->capture_stream);
  if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  if (c->aux_fork) cudaEventDestroy(c->aux_fork);
  if (c->aux_join) cudaEventDestroy(c->aux_join);
  delete c;
}

const char* lscat_last_error(const lscat_ctx* c) { return c ? c->err.c_str() : ""; }


lscat_status lscat_launch_count(const lscat_ctx* c, uint64_t* out) {
  if (!c || !out) return LSCAT_ERR_INVALID_ARG;
  *out = c->launches;
  return LSCAT_OK;
}

lscat_status lscat_comm_unique_id(void* out) {
  if (!out) return LSCAT_ERR_INVALID_ARG;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return LSCAT_ERR_NCCL;
  memcpy(out, &id, sizeof id);
  return LSCAT_OK;
}

lscat_status lscat_comm_init(lscat_ctx* c, const void* uid, int rank, int world) {
  LSCAT_CHECK_CTX(c);
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !uid))
    return fail(c, LSCAT_ERR_INVALID_ARG, "comm_init: rank %d world %d", rank, world);
  delete c->comm;
  c->comm = nullptr;
  c->rank = rank;
  c->world = world;
  if (world == 1) return LSCAT_OK;
  LSCAT_CUDA(c, cudaSetDevice(c->device));
  ncclUniqueId id;
  memcpy(&id, uid, sizeof id);
  ncclComm_t nc = nullptr;
  ncclResult_t r = ncclCommInitRank(&nc, world, id, rank);
  if (r != ncclSuccess) {
    c->world = 1;
    c->rank = 0;
    return fail(c, LSCAT_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  c->comm = make_nccl_comm(nc);
  return LSCAT_OK;
}

lscat_status lscat_comm_init_local(lscat_ctx* c, const char* name, int rank, int world) {
  LSCAT_CHECK_CTX(c);
  if (!name || world < 1 || rank < 0 || rank >= world)
    return fail(c, LSCAT_ERR_INVALID_ARG, "comm_init_local: rank %d world %d", rank, world);
  delete c->comm;
  c->comm = world > 1 ? make_local_comm(name, rank, world) : nullptr;
  c->rank = rank;
  c->world = world;
  return LSCAT_OK;
}

lscat_status lscat_kernel_work(uint32_t kernel, uint32_t n, uint64_t* bytes, uint64_t* flops) {
  if (!bytes || !flops || !kernel_table(kernel) || n == 0) return LSCAT_ERR_INVALID_ARG;
  kernel_work(kernel, n, bytes, flops);
  return LSCAT_OK;
}

// ---- a2: planner ---------------------------------------------------------------------
// Cost of one point (seconds): (W + K R) * max(bytes/BW, flops/peak, t_launch); points
// without an implementation (INVALID_CONFIG) cost nothing.  LPT: heaviest first, ties by
// lower id, onto the least-loaded rank, ties by lower rank.  (SURVEY §8(e).)
lscat_status lscat_plan(const lscat_plan_opts* o, int rank, int world, uint32_t* out,
                        uint64_t cap, uint64_t* n_out) {
  if (!o || !n_out || world < 1 || rank < 0 || rank >= world) return LSCAT_ERR_INVALID_ARG;
  if (!o->kernels || !o->sizes || o->n_kernels == 0 || o->n_sizes == 0) return LSCAT_ERR_INVALID_ARG;
  if (!block_list_ok(o->blocks, o->n_blocks)) return LSCAT_ERR_INVALID_ARG;
  if (o->shard != LSCAT_SHARD_POINT_LPT && o->shard != LSCAT_SHARD_GROUP) return LSCAT_ERR_INVALID_ARG;
  for (uint32_t i = 0; i < o->n_kernels; i++)
    if (!kernel_table(o->kernels[i])) return LSCAT_ERR_INVALID_ARG;
  for (uint32_t i = 0; i < o->n_sizes; i++)
    if (o->sizes[i] == 0 || (i && o->sizes[i] <= o->sizes[i - 1])) return LSCAT_ERR_INVALID_ARG;
  const double tl = o->launch_overhead_s > 0 ? o->launch_overhead_s : 2e-6;
  const double bw = o->hbm_bytes_per_s > 0 ? o->hbm_bytes_per_s : 6.55e12;
  const double tc = o->tensor_flops_per_s > 0 ? o->tensor_flops_per_s : 1.64e15;
  const double fp32 = 75e12;
  const double reps = (double)o->warmup + (double)o->brackets * o->launches_per_bracket;
  const uint64_t nb = o->n_blocks, npts = (uint64_t)o->n_kernels * o->n_sizes * nb;
  std::vector<double> cost(npts);
  for (uint64_t p = 0; p < npts; p++) {
    uint32_t k = o->kernels[p / (o->n_sizes * nb)];
    uint32_t n = o->sizes[(p / nb) % o->n_sizes];
    uint32_t bi = o->blocks[p % nb] / 32 - 1;
    uint64_t by, fl;
    kernel_work(k, n, &by, &fl);
    double peak = (k == LSCAT_K_GEMM_BF16) ? tc : fp32;
    double t = std::max({by / bw, fl / peak, tl});
    cost[p] = kernel_table(k)->fn[bi] ? reps * t : 0.0;
  }
  // units: points, or whole groups
  const bool by_group = o->shard == LSCAT_SHARD_GROUP;
  const uint64_t nunits = by_group ? npts / nb : npts;
  std::vector<double> ucost(nunits, 0.0);
  for (uint64_t p = 0; p < npts; p++) ucost[by_group ? p / nb : p] += cost[p];
  std::vector<uint64_t> order(nunits);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint64_t a, uint64_t b) { return ucost[a] > ucost[b]; });
  using Load = std::pair<double, int>;  // (load, rank): min-heap, ties -> lower rank
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (int r = 0; r < world; r++) heap.push({0.0, r});
  std::vector<int> owner(nunits);
  for (uint64_t u : order) {
    Load l = heap.top();
    heap.pop();
    owner[u] = l.second;
    heap.push({l.first + ucost[u], l.second});
  }
  uint64_t cnt = 0;
  for (uint64_t p = 0; p < npts; p++) cnt += owner[by_group ? p / nb : p] == rank;
  *n_out = cnt;
  if (!out) return LSCAT_OK;
  if (cnt > cap) return LSCAT_ERR_INVALID_ARG;  // nothing written
  uint64_t i = 0;
  for (uint64_t p = 0; p < npts; p++)
    if (owner[by_group ? p / nb : p] == rank) out[i++] = (uint32_t)p;
  return LSCAT_OK;
}

}  // extern "C"
