// sweep.cu — a4/a5: time every (kernel, N, block) point of this rank and emit the runtime table.
//
// Paper protocol: preheat once, launch the kernel 1000 times, repeat and take the
// median; Linux `timeout` turns hung / too-slow runs into NaN rows.  Here:
//   warm-up launches bracketed by events -> host waits -> predicted point time = warm * K * R;
//   over the timeout -> NaN + TIMEOUT without running the brackets;
//   otherwise K brackets of R launches, each bracket between two CUDA events on `stream`,
//   launched as pre-instantiated CUDA graphs (LSCAT_LAUNCH_GRAPH, chunks of <= 128 launches;
//   LSCAT_LAUNCH_GRAPH_PDL adds programmatic-dependent-launch edges between the captured
//   launches, so launch i+1 is scheduled and loads its read-only inputs while launch i
//   drains; every kernel still waits for its predecessor before its first global store)
//   or one cudaLaunchKernel per launch (LSCAT_LAUNCH_STREAM, the paper's host loop);
//   brackets are harvested lazily (one host wait per point, on the warm-up of the next one);
//   runtime = median over K of bracket/R; measured point time > timeout -> NaN + TIMEOUT.
// A kernel that never completes cannot be killed without losing the context: a host watchdog
// (polling cudaEventQuery) poisons the context after 4 x timeout + 30 s.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <thread>

#include "common.h"

namespace lscat {
namespace {

struct PointState {
  uint32_t p = 0;
  uint64_t row = 0;
  uint8_t status = LSCAT_ROW_OK;
  bool pending = false;  // brackets enqueued, not yet harvested
  double warm_ms = 0.0;  // total warm-up ms
  int slot = 0;
};

lscat_status wait_event(lscat_ctx* ctx, cudaEvent_t ev, double deadline_s) {
  auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    cudaError_t e = cudaEventQuery(ev);
    if (e == cudaSuccess) return LSCAT_OK;
    if (e != cudaErrorNotReady) return cuda_fail(ctx, e, "sweep: cudaEventQuery");
    double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > deadline_s) {
      ctx->poisoned = true;
      return fail(ctx, LSCAT_ERR_CUDA, "sweep watchdog: a launch did not complete within %.1f s", el);
    }
    if (el > 1e-3) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

cudaError_t get_graph(lscat_ctx* ctx, LaunchFn fn, const LaunchArgs& a, uint32_t kernel,
                      uint32_t n, uint32_t bi, uint32_t count, cudaGraphExec_t* out) {
  // the PDL flag is part of the key: the same point may be captured with and without it
  auto key = std::make_tuple(kernel, kernel == LSCAT_K_SPIN ? (uint32_t)a.spin_ns : n, bi,
                             count | (a.pdl ? 0x80000000u : 0u));
  auto it = ctx->graphs.find(key);
  if (it != ctx->graphs.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  cudaStream_t cs = ctx->capture_stream;
  cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return e;
  cudaError_t le = cudaSuccess;
  for (uint32_t i = 0; i < count && le == cudaSuccess; i++) le = fn(a, cs);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(cs, &g);
  if (le != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    return le;
  }
  if (e != cudaSuccess) return e;
  cudaGraphExec_t ex = nullptr;
  e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return e;
  ctx->graphs[key] = ex;
  *out = ex;
  return cudaSuccess;
}

}  // namespace
}  // namespace lscat

using namespace lscat;

extern "C" lscat_status lscat_sweep(lscat_ctx* ctx, const uint32_t* kernels, uint32_t nk,
                                    const uint32_t* sizes, uint32_t ns,
                                    const lscat_sweep_opts* o, lscat_table* out, void* stream) {
  LSCAT_CHECK_CTX(ctx);
  if (!o || !out || !kernels || !sizes || nk == 0 || ns == 0)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "sweep: null argument");
  if (!block_list_ok(o->blocks, o->n_blocks))
    return fail(ctx, LSCAT_ERR_INVALID_ARG,
                "sweep: blocks must be unique, ascending, multiples of 32 in [32, 1024] (P:98, P:215)");
  if (o->brackets == 0 || o->launches_per_bracket == 0 || !(o->timeout_s > 0))
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "sweep: brackets, launches_per_bracket, timeout_s must be > 0");
  if (o->launch_mode > LSCAT_LAUNCH_GRAPH_PDL || out->mem > LSCAT_MEM_HOST)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "sweep: bad launch_mode or table mem");
  if (!out->runtime_ms || !out->block_id || !out->group_offset)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "sweep: table needs runtime_ms, block_id, group_offset");
  for (uint32_t i = 0; i < nk; i++) {
    if (!kernel_table(kernels[i])) return fail(ctx, LSCAT_ERR_INVALID_ARG, "sweep: unknown kernel %u", kernels[i]);
    for (uint32_t j = 0; j < ns; j++)
      if (kernels[i] != LSCAT_K_SPIN && !ctx->suite.count({kernels[i], sizes[j]}))
        return fail(ctx, LSCAT_ERR_STATE, "sweep: (%u, %u) not registered", kernels[i], sizes[j]);
  }
  // ---- a2: plan
  lscat_plan_opts po{};
  po.kernels = kernels; po.n_kernels = nk; po.sizes = sizes; po.n_sizes = ns;
  po.blocks = o->blocks; po.n_blocks = o->n_blocks;
  po.warmup = o->warmup; po.brackets = o->brackets; po.launches_per_bracket = o->launches_per_bracket;
  po.shard = o->shard; po.launch_overhead_s = o->launch_overhead_s;
  uint64_t npts = 0;
  lscat_status st = lscat_plan(&po, ctx->rank, ctx->world, nullptr, 0, &npts);
  if (st) return fail(ctx, st, "sweep: plan rejected the options (sizes must be ascending)");
  std::vector<uint32_t> pts(npts);
  lscat_plan(&po, ctx->rank, ctx->world, pts.data(), npts, &npts);
  const uint64_t G = (uint64_t)nk * ns, nb = o->n_blocks;
  if (out->cap_rows < npts || out->cap_groups < G)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "sweep: table capacity %llu rows / %llu groups < %llu / %llu",
                (unsigned long long)out->cap_rows, (unsigned long long)out->cap_groups,
                (unsigned long long)npts, (unsigned long long)G);
  cudaStream_t s = (cudaStream_t)stream;
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));

  const uint32_t K = o->brackets, R = o->launches_per_bracket, W = o->warmup;
  const uint32_t chunk = std::min<uint32_t>(R, 128), full = R / chunk, rem = R % chunk;
  // event ring: per slot K+1 bracket events + 2 warm-up events
  constexpr int kRing = 32;
  const size_t evs_per = K + 3;
  while (ctx->events.size() < kRing * evs_per) {
    cudaEvent_t ev;
    LSCAT_CUDA(ctx, cudaEventCreate(&ev));
    ctx->events.push_back(ev);
  }
  auto EV = [&](int slot, size_t i) { return ctx->events[slot * evs_per + i]; };
  const double deadline = 4.0 * o->timeout_s + 30.0;

  std::vector<float> rt(npts, NAN);
  std::vector<uint16_t> bid(npts);
  std::vector<uint8_t> stat(npts, LSCAT_ROW_OK);
  std::vector<float> brk(o->bracket_ms_host ? npts * K : 0, NAN);
  std::vector<PointState> ring(kRing);
  std::vector<double> tmp(K);

  auto harvest = [&](PointState& ps) -> lscat_status {
    if (!ps.pending) return LSCAT_OK;
    ps.pending = false;
    lscat_status w = wait_event(ctx, EV(ps.slot, K), deadline);
    if (w) return w;
    double total = ps.warm_ms;
    for (uint32_t k = 0; k < K; k++) {
      float ms = 0.f;
      LSCAT_CUDA(ctx, cudaEventElapsedTime(&ms, EV(ps.slot, k), EV(ps.slot, k + 1)));
      tmp[k] = (double)ms / R;
      total += ms;
      if (!brk.empty()) brk[ps.row * K + k] = (float)tmp[k];
    }
    std::sort(tmp.begin(), tmp.end());
    double med = (K & 1) ? tmp[K / 2] : 0.5 * (tmp[K / 2 - 1] + tmp[K / 2]);
    if (total * 1e-3 > o->timeout_s) {
      stat[ps.row] = LSCAT_ROW_TIMEOUT;
      rt[ps.row] = NAN;
    } else {
      rt[ps.row] = (float)med;
    }
    return LSCAT_OK;
  };

  for (uint64_t i = 0; i < npts; i++) {
    const uint32_t p = pts[i];
    const uint32_t ki = p / (uint32_t)(ns * nb), si = (p / (uint32_t)nb) % ns, b = p % (uint32_t)nb;
    const uint32_t kern = kernels[ki], n = sizes[si], bi = o->blocks[b] / 32 - 1;
    bid[i] = (uint16_t)b;
    PointState& ps = ring[i % kRing];
    if ((st = harvest(ps))) return st;  // slot reuse: the point kRing back must be done
    ps = PointState{};
    ps.p = p;
    ps.row = i;
    ps.slot = (int)(i % kRing);
    LaunchFn fn = kernel_table(kern)->fn[bi];
    if (!fn) {
      stat[i] = LSCAT_ROW_INVALID_CONFIG;
      continue;
    }
    SuiteEntry dummy;
    const SuiteEntry* e = kern == LSCAT_K_SPIN ? &dummy : &ctx->suite[{kern, n}];
    LaunchArgs a{e, o->spin_ns};
    // warm-up (preheat)
    LSCAT_CUDA(ctx, cudaEventRecord(EV(ps.slot, K + 1), s));
    cudaError_t le = cudaSuccess;
    for (uint32_t w = 0; w < W && le == cudaSuccess; w++) le = fn(a, s);
    if (le != cudaSuccess) {
      if (is_sticky(le)) return cuda_fail(ctx, le, "sweep: warm-up launch");
      cudaGetLastError();
      stat[i] = (le == cudaErrorInvalidConfiguration || le == cudaErrorLaunchOutOfResources)
                    ? LSCAT_ROW_INVALID_CONFIG : LSCAT_ROW_LAUNCH_ERROR;
      continue;
    }
    ctx->launches += W;
    LSCAT_CUDA(ctx, cudaEventRecord(EV(ps.slot, K + 2), s));
    if ((st = wait_event(ctx, EV(ps.slot, K + 2), deadline))) return st;
    {
      cudaError_t ae = cudaGetLastError();
      if (ae != cudaSuccess) return cuda_fail(ctx, ae, "sweep: warm-up execution");
    }
    if (W > 0) {
      float ms = 0.f;
      LSCAT_CUDA(ctx, cudaEventElapsedTime(&ms, EV(ps.slot, K + 1), EV(ps.slot, K + 2)));
      ps.warm_ms = ms;
      const double predicted_s = (double)ms / W * K * R * 1e-3;
      if (predicted_s > o->timeout_s || ms * 1e-3 > o->timeout_s) {
        stat[i] = LSCAT_ROW_TIMEOUT;
        continue;
      }
    }
    // brackets
    cudaGraphExec_t gx = nullptr, gr = nullptr;
    const bool graph = o->launch_mode != LSCAT_LAUNCH_STREAM;
    if (graph) {
      LaunchArgs ga = a;
      ga.pdl = o->launch_mode == LSCAT_LAUNCH_GRAPH_PDL;
      le = get_graph(ctx, fn, ga, kern, n, bi, chunk, &gx);
      if (le == cudaSuccess && rem) le = get_graph(ctx, fn, ga, kern, n, bi, rem, &gr);
      if (le != cudaSuccess) {
        if (is_sticky(le)) return cuda_fail(ctx, le, "sweep: graph capture");
        cudaGetLastError();
        stat[i] = LSCAT_ROW_LAUNCH_ERROR;
        continue;
      }
    }
    LSCAT_CUDA(ctx, cudaEventRecord(EV(ps.slot, 0), s));
    for (uint32_t k = 0; k < K; k++) {
      if (graph) {
        for (uint32_t c = 0; c < full; c++) LSCAT_CUDA(ctx, cudaGraphLaunch(gx, s));
        if (rem) LSCAT_CUDA(ctx, cudaGraphLaunch(gr, s));
      } else {
        for (uint32_t r = 0; r < R; r++) {
          le = fn(a, s);
          if (le != cudaSuccess) return cuda_fail(ctx, le, "sweep: bracket launch");
        }
      }
      LSCAT_CUDA(ctx, cudaEventRecord(EV(ps.slot, k + 1), s));
    }
    ctx->launches += (uint64_t)K * R;
    ps.pending = true;
  }
  for (auto& ps : ring)
    if ((st = harvest(ps))) return st;

  // ---- a5: emit the table (groups in canonical order, rows ascending by block id)
  std::vector<int64_t> off(G + 1, 0);
  for (uint64_t i = 0; i < npts; i++) off[pts[i] / nb + 1]++;
  for (uint64_t g = 0; g < G; g++) off[g + 1] += off[g];
  std::vector<uint32_t> gk(G), gm(G);
  for (uint64_t g = 0; g < G; g++) {
    gk[g] = kernels[g / ns];
    gm[g] = (uint32_t)(g % ns);
  }
  if (out->mem == LSCAT_MEM_DEVICE) {
    auto h2d = cudaMemcpyHostToDevice;
    LSCAT_CUDA(ctx, cudaMemcpyAsync(out->runtime_ms, rt.data(), npts * 4, h2d, s));
    LSCAT_CUDA(ctx, cudaMemcpyAsync(out->block_id, bid.data(), npts * 2, h2d, s));
    if (out->status) LSCAT_CUDA(ctx, cudaMemcpyAsync(out->status, stat.data(), npts, h2d, s));
    LSCAT_CUDA(ctx, cudaMemcpyAsync(out->group_offset, off.data(), (G + 1) * 8, h2d, s));
    if (out->group_kernel) LSCAT_CUDA(ctx, cudaMemcpyAsync(out->group_kernel, gk.data(), G * 4, h2d, s));
    if (out->group_matrix) LSCAT_CUDA(ctx, cudaMemcpyAsync(out->group_matrix, gm.data(), G * 4, h2d, s));
    LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
  } else {
    memcpy(out->runtime_ms, rt.data(), npts * 4);
    memcpy(out->block_id, bid.data(), npts * 2);
    if (out->status) memcpy(out->status, stat.data(), npts);
    memcpy(out->group_offset, off.data(), (G + 1) * 8);
    if (out->group_kernel) memcpy(out->group_kernel, gk.data(), G * 4);
    if (out->group_matrix) memcpy(out->group_matrix, gm.data(), G * 4);
  }
  if (o->bracket_ms_host) memcpy(o->bracket_ms_host, brk.data(), brk.size() * 4);
  out->n_rows = npts;
  out->n_groups = G;
  out->rows_per_group = 0;
  out->first_group = 0;
  return LSCAT_OK;
}
