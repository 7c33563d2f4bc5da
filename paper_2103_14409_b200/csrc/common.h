// common.h — internal types of liblscat (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "comm.h"
#include "lscat.h"

namespace lscat {

constexpr int kMaxBlockIdx = 32;  // block sizes 32..1024 in steps of 32

// Device buffers of one registered (kernel, N) pair.
struct SuiteEntry {
  uint32_t kernel = 0, n = 0;
  void* in0 = nullptr;
  void* in1 = nullptr;
  void* out = nullptr;
  uint64_t in0_bytes = 0, in1_bytes = 0, out_bytes = 0;
  void* scratch = nullptr;  // colsum: partials + tile counters
  uint64_t scratch_bytes = 0;
  alignas(64) unsigned char host_blob[512] = {};  // gemm: the TMA tensor maps
};

struct LaunchArgs {
  const SuiteEntry* e;
  uint64_t spin_ns;
  bool pdl = false;  // programmatic dependent launch (LSCAT_LAUNCH_GRAPH_PDL); honoured only
                     // by kernels that call pdl_wait() before their first global store
  int sms = 148;     // SMs of the context's device (grid sizing; from lscat_ctx, not a static)
  size_t l2_bytes = 0;  // L2 size of the context's device (the row kernels' L2 keep share)
  bool cold = false;  // LSCAT_L2_ROTATE: no L2 keep policies (cold-HBM measurement)
};

// One launch of a suite kernel at block index bi (threads = 32*(bi+1)).  Returns the
// cudaGetLastError() of the launch (cudaSuccess on success).
using LaunchFn = cudaError_t (*)(const LaunchArgs&, cudaStream_t);

// Per-kernel dispatch: nullptr entries = no implementation at that block (INVALID_CONFIG).
// AttrFn gives the device function the default launch at that block size runs and its dynamic
// shared memory (raising the kernel's max-dynamic-smem attribute when needed), for the
// occupancy API in lscat_occupancy_block / lscat_kernel_attrs.
using AttrFn = cudaError_t (*)(const void** func, size_t* dyn_smem);

struct KernelTable {
  LaunchFn fn[kMaxBlockIdx];
  AttrFn attrs[kMaxBlockIdx];
};

// registries filled by each kernel translation unit
const KernelTable& table_euclid();
const KernelTable& table_matvec();
const KernelTable& table_rowsum();
const KernelTable& table_colsum();
const KernelTable& table_transpose();
const KernelTable& table_axpy();
const KernelTable& table_stencil5();
const KernelTable& table_gemm();
const KernelTable& table_spin();
const KernelTable* kernel_table(uint32_t kernel);

// suite buffer preparation that needs kernel-specific knowledge
cudaError_t colsum_prepare(SuiteEntry& e);
cudaError_t gemm_prepare(SuiteEntry& e);

// reducer scratch kept between lscat_reduce_table and lscat_stats
struct ReduceState {
  bool valid = false;
  lscat_reduce_opts opts{};
  uint64_t n_groups = 0;       // groups of the reduced table
  uint64_t own_lo = 0, own_hi = 0;  // groups whose values feed percentiles on this rank
  double* perf = nullptr;      // device [n_groups] (caller's or scratch)
  double* gain = nullptr;
  uint64_t* partials = nullptr;  // device, len = partials_len (SUM-merged)
  uint64_t* minmax = nullptr;    // device [4]: perf min, perf max, gain min, gain max keys
  // percentile selection already enqueued by lscat_reduce_table (opts.n_percentiles, R-27)
  uint32_t early = 0;            // EARLY_NONE / EARLY_SMALL / EARLY_SAMPLED
  // pinned host copy of the partials, enqueued by the reduce call (EARLY_SMALL; else null)
  const uint64_t* partials_h = nullptr;
  std::vector<double> early_pct;
};
enum { EARLY_NONE = 0, EARLY_SMALL = 1, EARLY_SAMPLED = 2 };

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace lscat

struct lscat_ctx {
  int device = 0;
  uint64_t seed = 0;
  bool poisoned = false;
  std::string err;
  int sm_count = 0;
  uint64_t launches = 0;  // device kernels launched (lscat_launch_count)
  size_t l2_bytes = 0;
  // suite
  std::map<std::pair<uint32_t, uint32_t>, lscat::SuiteEntry> suite;
  // graphs: (kernel, n, block_idx, chunk) -> exec
  std::map<std::tuple<uint32_t, uint32_t, uint32_t, uint32_t>, cudaGraphExec_t> graphs;
  cudaStream_t capture_stream = nullptr;
  // side branch of a reduce call (the host copy of the partials next to the early selection)
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
  // percentile selection: first batch (init + 3 levels + state read-back) as a graph, keyed by
  // every pointer / size / percentile it bakes in (stats.cu; world == 1)
  std::vector<std::pair<std::string, cudaGraphExec_t>> sel_graphs;
  // lscat_reduce_table on small device tables (one rank): everything it enqueues as one cached
  // graph, keyed by its arguments; valid while no scratch / pinned buffer was (re)allocated
  struct RedGraph {
    std::string key;
    cudaGraphExec_t gx = nullptr;  // null: seen once (captured on the next call) or not capturable
    bool tried = false;        // a capture was attempted
    uint64_t gen = 0;          // scratch_gen at capture
    lscat::ReduceState rs;     // the context state the call leaves
    uint64_t launches = 0;     // kernels one call launches
  };
  std::vector<RedGraph> red_graphs;
  uint64_t scratch_gen = 0;    // bumped by every scratch / pinned (re)allocation
  // kernel attributes / occupancy already set or queried on this context's device (host calls
  // kept off the launch path of the small tables)
  std::map<std::pair<bool, size_t>, int> red_occ;
  int sel_occ0 = 0, sel_occ1 = 0;
  uint64_t sel_fallbacks = 0;  // sampled first levels that missed a target (stats.cu)
  uint64_t fin_fallbacks = 0;  // sel_finish runs that handed over to the chain (stats.cu)
  std::vector<cudaEvent_t> events;
  // LSCAT_L2_ROTATE (sweep.cu): the (kernel, n) whose input copies the "rot" scratch arena
  // holds, and the arena base its graphs were captured against
  std::pair<uint32_t, uint32_t> rot_owner{~0u, ~0u};
  void* rot_base = nullptr;
  // comm
  lscat::Comm* comm = nullptr;  // NCCL, or the local test transport (comm.h)
  int rank = 0, world = 1;
  // reducer scratch
  lscat::ReduceState rs;
  std::map<std::string, lscat::DevBuf> scratch;
  std::map<std::string, lscat::DevBuf> pinned;  // cudaMallocHost staging
};

namespace lscat {

// error helpers ---------------------------------------------------------------------------
lscat_status fail(lscat_ctx* ctx, lscat_status s, const char* fmt, ...);
lscat_status cuda_fail(lscat_ctx* ctx, cudaError_t e, const char* what);
bool is_sticky(cudaError_t e);
// device scratch (grow-only) keyed by name
void* scratch(lscat_ctx* ctx, const char* name, size_t bytes, cudaError_t* err);
// pinned host staging (grow-only) keyed by name
void* pinned(lscat_ctx* ctx, const char* name, size_t bytes, cudaError_t* err);
// Raise a kernel's max-dynamic-shared-memory attribute on the current device to at least
// `bytes` (device-global state: never lowered, set once per (kernel, device, size increase)).
cudaError_t ensure_smem_attr(const void* func, size_t bytes);
constexpr uint64_t kEarlySmallGroups = 1ull << 20;  // = stats.cu kSmallKeys (one-launch selection)
// percentile selection enqueued by lscat_reduce_table (stats.cu; R-27), no host sync: the
// one-launch selection (small tables) or the sampled first level + sel_finish (large tables)
// on the kept per-group values; *kind = EARLY_NONE when this device / percentile list cannot
lscat_status early_select(lscat_ctx* ctx, const double* perf, const double* gain, uint64_t lo, uint64_t hi,
                          const uint64_t* partials, const uint64_t* mm, uint32_t nb, const double* pct,
                          uint32_t npct, cudaStream_t s, uint32_t* kind);
// host-side work model
void kernel_work(uint32_t kernel, uint32_t n, uint64_t* bytes, uint64_t* flops);
bool block_list_ok(const uint16_t* blocks, uint32_t n);

}  // namespace lscat

#define LSCAT_CHECK_CTX(ctx)                                                        \
  do {                                                                              \
    if (!(ctx)) return LSCAT_ERR_INVALID_ARG;                                       \
    if ((ctx)->poisoned) return LSCAT_ERR_CUDA;                                     \
  } while (0)

#define LSCAT_CUDA(ctx, call)                                                       \
  do {                                                                              \
    cudaError_t e__ = (call);                                                       \
    if (e__ != cudaSuccess) return lscat::cuda_fail((ctx), e__, #call);             \
  } while (0)
