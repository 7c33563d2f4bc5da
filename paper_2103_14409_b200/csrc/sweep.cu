// sweep.cu — a4/a5: time every (kernel, N, block) point of this rank and emit the runtime table.
//
// Paper protocol: preheat once, launch the kernel 1000 times, repeat and take the
// median; Linux `timeout` turns hung / too-slow runs into NaN rows.  Here:
//   warm-up launches bracketed by events -> host waits -> predicted point time = warm * K * R;
//   over the timeout -> NaN + TIMEOUT without running the brackets; without a prediction, or
//   one above half the budget, the brackets are issued one at a time (one queued ahead) and
//   the point stops as soon as the elapsed time or first bracket x K exceeds the budget;
//   brackets are timed by CUDA events or by %globaltimer stamp kernels (lscat_timer);
//   LSCAT_L2_ROTATE cycles copies of the point's buffers launch by launch (cold L2);
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
  bool pending = false;  // brackets enqueued, not yet harvested
  double warm_ms = 0.0;  // total warm-up ms
  int slot = 0;
  uint32_t nk = 0;       // brackets enqueued (< K: the budget stopped the point, A-18)
};

// %globaltimer stamp (ns) written by one thread: the GLOBALTIMER bracket clock.
__global__ void stamp_kernel(unsigned long long* __restrict__ dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

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

constexpr uint32_t kKeyPdl = 0x80000000u, kKeyRot = 0x40000000u;

// A graph of `count` back-to-back launches; launch i uses args[i % nargs] (ROTATE cycles the
// buffer copies).  Cached per (kernel, n, block, count, pdl, rotate).
cudaError_t get_graph(lscat_ctx* ctx, LaunchFn fn, const LaunchArgs* args, uint32_t nargs,
                      uint32_t kernel, uint32_t n, uint32_t bi, uint32_t count, bool rot,
                      cudaGraphExec_t* out) {
  const LaunchArgs& a = args[0];
  auto key = std::make_tuple(kernel, kernel == LSCAT_K_SPIN ? (uint32_t)a.spin_ns : n, bi,
                             count | (a.pdl ? kKeyPdl : 0u) | (rot ? kKeyRot : 0u));
  auto it = ctx->graphs.find(key);
  if (it != ctx->graphs.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  cudaStream_t cs = ctx->capture_stream;
  cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return e;
  cudaError_t le = cudaSuccess;
  for (uint32_t i = 0; i < count && le == cudaSuccess; i++) le = fn(args[i % nargs], cs);
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

// LSCAT_L2_ROTATE: c copies of (kernel, n)'s buffers in the ctx arena (scratch "rot"), c =
// clamp(ceil(2 L2 / footprint), 2, 128).  Inputs are copied from the registered entry when
// the arena last held another pair (stream-ordered after the previous point's launches; not
// timed).  The copies share the original's kernel scratch (colsum partials/tickets: launches
// are serialised).  Graphs captured over an arena that is reallocated are dropped.
lscat_status rotate_setup(lscat_ctx* ctx, const SuiteEntry& e, cudaStream_t s,
                          std::vector<SuiteEntry>& ents) {
  auto up = [](uint64_t b) { return (b + 255) & ~255ull; };
  const uint64_t F = up(e.in0_bytes) + up(e.in1_bytes) + up(e.out_bytes);
  const uint64_t want = F ? (2ull * ctx->l2_bytes + F - 1) / F : 2;
  const uint32_t c = (uint32_t)std::min<uint64_t>(128, std::max<uint64_t>(2, want));
  cudaError_t err = cudaSuccess;
  uint8_t* base = (uint8_t*)scratch(ctx, "rot", c * F, &err);
  if (err != cudaSuccess) return cuda_fail(ctx, err, "sweep: rotation arena");
  if (base != ctx->rot_base) {
    for (auto it = ctx->graphs.begin(); it != ctx->graphs.end();) {
      if (std::get<3>(it->first) & kKeyRot) {
        cudaGraphExecDestroy(it->second);
        it = ctx->graphs.erase(it);
      } else {
        ++it;
      }
    }
    ctx->rot_base = base;
    ctx->rot_owner = {~0u, ~0u};
  }
  const bool copy = ctx->rot_owner != std::make_pair(e.kernel, e.n);
  ents.assign(c, e);
  for (uint32_t i = 0; i < c; i++) {
    SuiteEntry& x = ents[i];
    uint8_t* b = base + (uint64_t)i * F;
    x.in0 = e.in0 ? b : nullptr;
    x.in1 = e.in1 ? b + up(e.in0_bytes) : nullptr;
    x.out = e.out ? b + up(e.in0_bytes) + up(e.in1_bytes) : nullptr;
    if (copy) {
      if (e.in0) LSCAT_CUDA(ctx, cudaMemcpyAsync(x.in0, e.in0, e.in0_bytes, cudaMemcpyDeviceToDevice, s));
      if (e.in1) LSCAT_CUDA(ctx, cudaMemcpyAsync(x.in1, e.in1, e.in1_bytes, cudaMemcpyDeviceToDevice, s));
    }
    if (e.kernel == LSCAT_K_GEMM_BF16 && (err = gemm_prepare(x)) != cudaSuccess)
      return cuda_fail(ctx, err, "sweep: rotation tensor maps");
  }
  ctx->rot_owner = {e.kernel, e.n};
  return LSCAT_OK;
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
  if (o->timer > LSCAT_TIMER_GLOBALTIMER || o->l2_mode > LSCAT_L2_ROTATE || o->verify > 1)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "sweep: bad timer, l2_mode or verify");
  if (o->verify && (!o->verify_host || !o->verify_offsets))
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "sweep: verify needs verify_host and verify_offsets");
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
  auto point_kernel = [&](uint32_t p) { return kernels[p / (uint32_t)(ns * nb)]; };
  auto point_size = [&](uint32_t p) { return sizes[(p / (uint32_t)nb) % ns]; };
  // verify: every row reserves its point's output bytes (rows without a result stay unwritten)
  std::vector<uint64_t> voff;
  if (o->verify) {
    voff.assign(npts + 1, 0);
    for (uint64_t i = 0; i < npts; i++) {
      const uint32_t k = point_kernel(pts[i]);
      voff[i + 1] = voff[i] + (k == LSCAT_K_SPIN ? 0 : ctx->suite[{k, point_size(pts[i])}].out_bytes);
    }
    if (voff[npts] > o->verify_cap_bytes)
      return fail(ctx, LSCAT_ERR_INVALID_ARG, "sweep: verify needs %llu bytes, capacity %llu",
                  (unsigned long long)voff[npts], (unsigned long long)o->verify_cap_bytes);
  }
  cudaStream_t s = (cudaStream_t)stream;
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));

  const uint32_t K = o->brackets, R = o->launches_per_bracket, W = o->warmup;
  const bool gtimer = o->timer == LSCAT_TIMER_GLOBALTIMER;
  const bool rotate = o->l2_mode == LSCAT_L2_ROTATE;
  // event ring: per slot K+1 bracket events + 2 warm-up events
  constexpr int kRing = 32;
  const size_t evs_per = K + 3;
  while (ctx->events.size() < kRing * evs_per) {
    cudaEvent_t ev;
    LSCAT_CUDA(ctx, cudaEventCreate(&ev));
    ctx->events.push_back(ev);
  }
  auto EV = [&](int slot, size_t i) { return ctx->events[slot * evs_per + i]; };
  // globaltimer stamps: device [kRing][K+1], copied to pinned host after each point's brackets
  unsigned long long *stamp_d = nullptr, *stamp_h = nullptr;
  if (gtimer) {
    cudaError_t err = cudaSuccess;
    stamp_d = (unsigned long long*)scratch(ctx, "stamps", kRing * (K + 1) * 8, &err);
    if (err) return cuda_fail(ctx, err, "sweep: stamp buffer");
    stamp_h = (unsigned long long*)pinned(ctx, "stamps", kRing * (K + 1) * 8, &err);
    if (err) return cuda_fail(ctx, err, "sweep: pinned stamp buffer");
  }
  auto stamp = [&](int slot, uint32_t k) -> cudaError_t {
    stamp_kernel<<<1, 32, 0, s>>>(stamp_d + (size_t)slot * (K + 1) + k);
    ctx->launches++;
    return cudaGetLastError();
  };
  // one untimed stamp first: the kernel's (lazy) module load must not fall inside a bracket
  if (gtimer) LSCAT_CUDA(ctx, stamp(0, 0));
  const double deadline = 4.0 * o->timeout_s + 30.0;

  std::vector<float> rt(npts, NAN);
  std::vector<uint16_t> bid(npts);
  std::vector<uint8_t> stat(npts, LSCAT_ROW_OK);
  std::vector<float> brk(o->bracket_ms_host ? npts * K : 0, NAN);
  std::vector<float> brk_ev(o->bracket_ms_event_host ? npts * K : 0, NAN);
  std::vector<PointState> ring(kRing);
  std::vector<double> tmp(K);

  auto ev_ms = [&](int slot, size_t a, size_t b, double* ms) -> lscat_status {
    float f = 0.f;
    LSCAT_CUDA(ctx, cudaEventElapsedTime(&f, EV(slot, a), EV(slot, b)));
    *ms = f;
    return LSCAT_OK;
  };
  auto harvest = [&](PointState& ps) -> lscat_status {
    if (!ps.pending) return LSCAT_OK;
    ps.pending = false;
    // with GLOBALTIMER the stamps' copy to the host follows the last bracket's event: wait for
    // the event recorded after that copy (reading the pinned stamps earlier raced with the copy)
    lscat_status w = wait_event(ctx, EV(ps.slot, gtimer ? K + 2 : ps.nk), deadline);
    if (w) return w;
    double total = ps.warm_ms;
    const unsigned long long* sh = gtimer ? stamp_h + (size_t)ps.slot * (K + 1) : nullptr;
    for (uint32_t k = 0; k < ps.nk; k++) {
      double ms = 0.0;
      if ((w = ev_ms(ps.slot, k, k + 1, &ms))) return w;
      total += ms;
      const double gms = gtimer ? (double)(sh[k + 1] - sh[k]) * 1e-6 : ms;
      tmp[k] = gms / R;
      if (!brk.empty()) brk[ps.row * K + k] = (float)tmp[k];
      if (!brk_ev.empty()) brk_ev[ps.row * K + k] = (float)(ms / R);
    }
    if (ps.nk < K || total * 1e-3 > o->timeout_s) {  // budget exceeded (A-18)
      stat[ps.row] = LSCAT_ROW_TIMEOUT;
      rt[ps.row] = NAN;
      return LSCAT_OK;
    }
    std::sort(tmp.begin(), tmp.begin() + K);
    rt[ps.row] = (float)((K & 1) ? tmp[K / 2] : 0.5 * (tmp[K / 2 - 1] + tmp[K / 2]));
    return LSCAT_OK;
  };

  std::vector<SuiteEntry> rot_ents;
  std::vector<LaunchArgs> args;
  for (uint64_t i = 0; i < npts; i++) {
    const uint32_t p = pts[i];
    const uint32_t b = p % (uint32_t)nb;
    const uint32_t kern = point_kernel(p), n = point_size(p), bi = o->blocks[b] / 32 - 1;
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
    a.sms = ctx->sm_count;
    a.l2_bytes = ctx->l2_bytes;
    a.cold = rotate;
    a.pdl = false;
    args.assign(1, a);
    if (rotate && kern != LSCAT_K_SPIN) {
      if ((st = rotate_setup(ctx, *e, s, rot_ents))) return st;
      args.resize(rot_ents.size(), a);
      for (size_t c = 0; c < rot_ents.size(); c++) args[c].e = &rot_ents[c];
    }
    const uint32_t nargs = (uint32_t)args.size();
    // warm-up (preheat)
    LSCAT_CUDA(ctx, cudaEventRecord(EV(ps.slot, K + 1), s));
    cudaError_t le = cudaSuccess;
    for (uint32_t w = 0; w < W && le == cudaSuccess; w++) le = fn(args[w % nargs], s);
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
    double predicted_s = -1.0;
    if (W > 0) {
      double ms = 0.0;
      if ((st = ev_ms(ps.slot, K + 1, K + 2, &ms))) return st;
      ps.warm_ms = ms;
      predicted_s = ms / W * K * R * 1e-3;
      if (predicted_s > o->timeout_s || ms * 1e-3 > o->timeout_s) {
        stat[i] = LSCAT_ROW_TIMEOUT;
        continue;
      }
    }
    // no prediction, or one close to the budget: check the budget after every bracket
    const bool careful = predicted_s < 0.0 || predicted_s > 0.5 * o->timeout_s;
    // brackets
    cudaGraphExec_t gx = nullptr, gr = nullptr;
    const bool graph = o->launch_mode != LSCAT_LAUNCH_STREAM;
    // graph chunks of <= 128 launches; with ROTATE a whole number of copy cycles
    uint32_t chunk = std::min<uint32_t>(R, 128);
    if (nargs > 1) chunk = std::min<uint32_t>(R, nargs * std::max<uint32_t>(1, 128 / nargs));
    const uint32_t full = R / chunk, rem = R % chunk;
    if (graph) {
      for (auto& x : args) x.pdl = o->launch_mode == LSCAT_LAUNCH_GRAPH_PDL;
      le = get_graph(ctx, fn, args.data(), nargs, kern, n, bi, chunk, nargs > 1, &gx);
      if (le == cudaSuccess && rem) le = get_graph(ctx, fn, args.data(), nargs, kern, n, bi, rem, nargs > 1, &gr);
      if (le != cudaSuccess) {
        if (is_sticky(le)) return cuda_fail(ctx, le, "sweep: graph capture");
        cudaGetLastError();
        stat[i] = LSCAT_ROW_LAUNCH_ERROR;
        continue;
      }
    }
    LSCAT_CUDA(ctx, cudaEventRecord(EV(ps.slot, 0), s));
    if (gtimer) LSCAT_CUDA(ctx, stamp(ps.slot, 0));
    uint32_t k = 0;
    for (; k < K; k++) {
      if (careful && k >= 2) {  // bracket k-2 done (k-1 still queued): elapsed and prediction
        if ((st = wait_event(ctx, EV(ps.slot, k - 1), deadline))) return st;
        double el = ps.warm_ms, first = 0.0;
        for (uint32_t j = 0; j + 1 < k; j++) {
          double ms = 0.0;
          if ((st = ev_ms(ps.slot, j, j + 1, &ms))) return st;
          el += ms;
          if (j == 0) first = ms;
        }
        if (el * 1e-3 > o->timeout_s || first * K * 1e-3 > o->timeout_s) break;  // skip the rest
      }
      if (graph) {
        for (uint32_t c = 0; c < full; c++) LSCAT_CUDA(ctx, cudaGraphLaunch(gx, s));
        if (rem) LSCAT_CUDA(ctx, cudaGraphLaunch(gr, s));
      } else {
        for (uint32_t r = 0; r < R; r++) {
          le = fn(args[r % nargs], s);
          if (le != cudaSuccess) return cuda_fail(ctx, le, "sweep: bracket launch");
        }
      }
      LSCAT_CUDA(ctx, cudaEventRecord(EV(ps.slot, k + 1), s));
      if (gtimer) LSCAT_CUDA(ctx, stamp(ps.slot, k + 1));
    }
    ps.nk = k;
    ctx->launches += (uint64_t)k * R;
    if (gtimer) {
      LSCAT_CUDA(ctx, cudaMemcpyAsync(stamp_h + (size_t)ps.slot * (K + 1), stamp_d + (size_t)ps.slot * (K + 1),
                                      (size_t)(k + 1) * 8, cudaMemcpyDeviceToHost, s));
      // EV(K + 2) (the warm-up's end, already waited for above) now marks the copy's completion
      LSCAT_CUDA(ctx, cudaEventRecord(EV(ps.slot, K + 2), s));
    }
    if (o->verify && k == K && kern != LSCAT_K_SPIN) {  // the last timed launch's output
      const SuiteEntry* last = args[(R - 1) % nargs].e;
      LSCAT_CUDA(ctx, cudaMemcpyAsync((uint8_t*)o->verify_host + voff[i], last->out, last->out_bytes,
                                      cudaMemcpyDeviceToHost, s));
    }
    ps.pending = true;
  }
  for (auto& ps : ring)
    if ((st = harvest(ps))) return st;
  LSCAT_CUDA(ctx, cudaStreamSynchronize(s));  // verify copies

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
  if (o->bracket_ms_event_host) memcpy(o->bracket_ms_event_host, brk_ev.data(), brk_ev.size() * 4);
  if (o->verify) memcpy(o->verify_offsets, voff.data(), voff.size() * 8);
  out->n_rows = npts;
  out->n_groups = G;
  out->rows_per_group = 0;
  out->first_group = 0;
  return LSCAT_OK;
}
