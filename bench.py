#!/usr/bin/env python
"""Benchmark of the LS-CAT hot path on B200 (BASELINE.json metric: sweep points/s and table
rows/s; % HBM peak per kernel).

A step = one pass of the whole hot path over the configs[1] workload:
plan (a2) -> sweep `euclidean_kernel` over blocks 32..1024 step 32 x N = 64..8192 (a3-a5,
paper timing policy: 1 preheat + 10 brackets x 1000 launches, median; plain CUDA-graph
brackets, each launch waits for the previous one as in the paper's serial loop; warm L2 = the
paper's runtime definition) -> reduce the runtime table (a6/a7, NCCL merge a9 when N > 1) ->
stats with percentiles (a8/a10) -> the dominant point (euclid N = 8192 at the step's best
block) re-timed with cold L2 (LSCAT_L2_ROTATE) for the roofline.
`value` = sweep points/s of the whole job (points of all ranks / max-over-ranks device time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--policy paper|fast]
                    [--launch graph|graph_pdl|stream] [--timer event|globaltimer]
                    [--impl ours|reference]

Multi-GPU: launched by torchrun, one rank per GPU, points LPT-sharded (strong scaling: the
256-point sweep is fixed); table rows/s of configs[2]-[4] sharded over the ranks (group-aligned
and point-sharded, NCCL merge).  `--impl reference` times the CPU oracle (the tier's reference
arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SIZES = [64, 128, 256, 512, 1024, 2048, 4096, 8192]
BLOCKS = list(range(32, 1025, 32))
POLICIES = {"paper": (1, 10, 1000), "fast": (1, 5, 20), "tiny": (1, 2, 2)}  # (W, K, R): P:203; tiny = ncu launch lists
METRIC = "sweep points/s (euclidean_kernel, 32 blocks x 8 matrix sizes)"
PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]


def env_int(k, d):
    return int(os.environ.get(k, d))


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p.get("bf16_tflops"), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            c = [x.strip() for x in line.split(",")]
            if len(c) < 9:
                continue
            try:
                sm.append(float(c[1]))
                mx.append(float(c[2]))
            except ValueError:
                continue
            for n, v in zip(names, c[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------
# reference arm: the CPU oracle (tier framing: the oracle is the reference)
# ----------------------------------------------------------------------------------------
def host_info():
    """Host cores this process may use and the CPU model (recorded with the
    CPU baseline)."""
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": cores, "cpu_count": os.cpu_count(), "cpu_model": model}


def _euclid_threads(OK, A, q, threads):
    """The oracle's fp64 euclid on row chunks in `threads` threads (numpy releases the GIL in
    its array kernels); the arithmetic per row is the oracle's own."""
    if threads <= 1 or A.shape[0] < 256:
        return OK.euclid(A, q)
    from concurrent.futures import ThreadPoolExecutor
    parts = np.array_split(np.arange(A.shape[0]), threads)
    with ThreadPoolExecutor(threads) as ex:
        return np.concatenate(list(ex.map(lambda ix: OK.euclid(A[ix[0]:ix[-1] + 1], q), parts)))


def oracle_points_per_s(policy, A_by_n=None, min_s=10.0, threads=1):
    """Time the fp64 oracle of euclidean_kernel on a bounded sample and scale to the policy:
    a point = (W + K*R) evaluations of the kernel at its N; 32 points per size.  The sample
    evaluates every matrix size once per round, for as many rounds as fit in `min_s` seconds
    of CPU work (at least one); the per-size time is the mean over rounds."""
    from oracle import kernels as OK
    W, K, R = POLICIES[policy]
    rng = np.random.default_rng(0)
    if A_by_n is None:
        A_by_n = {n: (rng.uniform(-1, 1, (n, n)).astype(np.float32),
                      rng.uniform(-1, 1, n).astype(np.float32)) for n in SIZES}
    per_n = {n: 0.0 for n in SIZES}
    rounds, work = 0, 0.0
    while rounds == 0 or work < min_s:
        for n in SIZES:
            A, q = A_by_n[n]
            t0 = time.perf_counter()
            _euclid_threads(OK, A, q, threads)
            dt = time.perf_counter() - t0
            per_n[n] += dt
            work += dt
        rounds += 1
    total = sum(len(BLOCKS) * (W + K * R) * per_n[n] / rounds for n in SIZES)
    return len(SIZES) * len(BLOCKS) / total, work, rounds


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    W, K = args.warmup, args.steps
    hi = host_info()
    rng = np.random.default_rng(0)
    A_by_n = {n: (rng.uniform(-1, 1, (n, n)).astype(np.float32),
                  rng.uniform(-1, 1, n).astype(np.float32)) for n in SIZES}
    for _ in range(W):
        oracle_points_per_s(args.policy, A_by_n, min_s=0.0)
    vals, cpu_s, rounds = [], 0.0, 0
    t0 = time.perf_counter()
    for _ in range(K):
        v, w, r = oracle_points_per_s(args.policy, A_by_n, min_s=5.0)
        vals.append(v)
        cpu_s += w
        rounds += r
    wall = time.perf_counter() - t0
    value = len(SIZES) * len(BLOCKS) * K / sum(len(SIZES) * len(BLOCKS) / v for v in vals)
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": args.gpus, "steps": K, "warmup": W, "ms_per_step": wall * 1e3 / K,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": "configs[1] euclid full sweep",
                                        "policy": args.policy, "blocks": "32..1024 step 32",
                                        "sizes": SIZES},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": 1, "kind": "oracle",
                         "host": hi,
                         "sample": f"per step: fp64 numpy evaluations of euclidean_kernel, "
                                   f"every matrix size once per round, rounds for >= 5 s of CPU "
                                   f"({rounds} rounds, {cpu_s:.1f} s in total), scaled by 32 blocks "
                                   f"x (W+K*R) launches per point"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


# ----------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--policy", choices=list(POLICIES), default="paper")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--launch", choices=["graph", "graph_pdl", "stream"], default="graph",
                    help="how a bracket's launches are issued (lscat_launch_mode); the runtime "
                         "table's default is plain graphs (launches serialised as in the paper)")
    ap.add_argument("--timer", choices=["event", "globaltimer"], default="event")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2103_14409_b200 as L

    rank, world, lrank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(lrank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    uid = [L.comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    ctx = L.Ctx(lrank, seed=0x15CA7)
    ctx.comm_init(uid[0], rank, world)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    W, K, R = POLICIES[args.policy]
    modes = {"graph": L.LAUNCH_GRAPH, "graph_pdl": L.LAUNCH_GRAPH_PDL, "stream": L.LAUNCH_STREAM}
    launch_mode = modes[args.launch]
    timer = {"event": L.TIMER_EVENT, "globaltimer": L.TIMER_GLOBALTIMER}[args.timer]
    ks = [L.K_EUCLID]
    ctx.register_suite(ks, SIZES)
    npts_total = len(ks) * len(SIZES) * len(BLOCKS)
    table = L.Table.empty(npts_total, len(ks) * len(SIZES))
    ropts = L.reduce_opts(len(BLOCKS), len(SIZES), point_sharded=1 if world > 1 else 0)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    g8 = len(SIZES) - 1
    # cold re-timing of the dominant point: W, K, R (scaled down with the policy so a tiny-policy
    # launch list under ncu keeps the sweep's proportions)
    COLD = {"paper": (1, 3, 200), "fast": (1, 3, 20), "tiny": (1, 1, 2)}[args.policy]

    def step(mode=launch_mode):
        t = ctx.sweep(ks, SIZES, BLOCKS, warmup=W, brackets=K, launches=R, timeout_s=30.0,
                      table=table, with_brackets=True, launch_mode=mode, timer=timer)
        red = ctx.reduce_table(t, ropts, per_group=True)
        st = ctx.stats(ropts, percentiles=PCTS)
        # the dominant kernel (euclid N = 8192) at the step's best block, cold L2: the roofline
        bb = int(red["best_block_id"][g8].item()) & 0xFFFF
        cold = None
        if bb < len(BLOCKS):
            c = ctx.sweep(ks, [8192], [BLOCKS[bb]], warmup=COLD[0], brackets=COLD[1],
                          launches=COLD[2], l2_mode=L.L2_ROTATE, with_brackets=True,
                          timer=timer, table=L.Table.empty(1, 1))
            cold = (BLOCKS[bb], c.brackets[0].copy() if c.n_rows else None)
        return t, st, red, cold

    for _ in range(args.warmup):
        step()
    barrier()
    clocks = Clocks(lrank)
    l0 = ctx.launch_count()
    dev_ms = 0.0
    brackets_all = []
    colds = []
    last = None
    for _ in range(args.steps):
        flush.zero_()                      # L2 flushed between timed steps (outside the events)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t, st, red, cold = step()
        e1.record(stream)
        barrier()
        dev_ms += e0.elapsed_time(e1)
        last = (t, st, red)
        brackets_all.append(t.brackets.copy())
        colds.append(cold)
    ck = clocks.stop()
    launches = ctx.launch_count() - l0
    tot_ms = allmax(dev_ms)
    value = npts_total * args.steps / (tot_ms / 1e3)

    # ---- roofline of the dominant kernel: euclidean_kernel at N = 8192, best block, cold L2
    tab = last[0].to_numpy()
    hbm_peak, tc_peak, peak_kind = load_peaks()
    nbytes, _ = L.kernel_work(L.K_EUCLID, 8192)
    lo, hi = tab["group_offset"][g8], tab["group_offset"][g8 + 1]
    roof, roof_warm = None, None
    cold_ms = [float(np.mean(c[1])) for c in colds if c and c[1] is not None and np.isfinite(c[1]).all()]
    if cold_ms:
        mean_ms = float(np.mean(cold_ms))
        achieved = nbytes / (mean_ms * 1e-3) / 1e9
        trs = load_traffic()  # the capture of the timed block when there is one
        tr = trs.get(f"euclid_8192_b{colds[-1][0]}_cold", trs.get("euclid_8192_cold"))
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": tr,
                "kernel": f"euclid N=8192 block={colds[-1][0]}", "peak_kind": peak_kind,
                "l2": "cold (LSCAT_L2_ROTATE: 2 buffer copies cycled, no L2 keep policy)",
                "algorithmic_bytes_per_launch": nbytes, "avg_launch_ms": round(mean_ms, 5),
                "timing": f"CUDA events ({args.timer}) over {COLD[1]} brackets x {COLD[2]} launches "
                          f"per timed step, inside the timed region"}
    if hi > lo:
        rt = tab["runtime_ms"][lo:hi]
        i = int(np.nanargmin(rt))
        mean_w = float(np.mean([b[lo + i].mean() for b in brackets_all]))
        share = sum(float(np.mean([b[lo + j].mean() for b in brackets_all]))
                    for j in range(hi - lo)) * (W + K * R) / (dev_ms / args.steps)
        tr = load_traffic().get("euclid_8192")
        roof_warm = {"kernel": f"euclid N=8192 block={BLOCKS[tab['block_id'][lo + i]]}",
                     "l2": "warm (the paper's loop: same buffers; the row kernel keeps a fraction "
                           "of A L2-resident across the bracket's launches)",
                     "avg_launch_ms": round(mean_w, 5),
                     "effective_gbs": round(nbytes / (mean_w * 1e-3) / 1e9, 1),
                     "effective_frac": round(nbytes / (mean_w * 1e-3) / 1e9 / hbm_peak, 4),
                     "share_of_step": round(share, 4)}
        if tr:
            roof_warm["dram_bytes_per_launch_steady"] = tr
            roof_warm["dram_frac"] = round(tr / (mean_w * 1e-3) / 1e9 / hbm_peak, 4)
        if roof:
            roof["share_of_step"] = roof_warm["share_of_step"]
    per_n = {}
    for gi, n in enumerate(SIZES):
        a, b = tab["group_offset"][gi], tab["group_offset"][gi + 1]
        if b > a:
            v = tab["runtime_ms"][a:b] * 1e3
            per_n[str(n)] = [round(float(np.nanmin(v)), 2), round(float(np.nanmedian(v)), 2),
                             round(float(np.nanmax(v)), 2)]
            if n >= 4096:
                per_n[f"{n}_by_block"] = [round(float(x), 1) for x in v]
    # SURVEY 8(d) sweep-point roofline: t_min(point) = (W + K R) max(bytes / BW, flops / TC,
    # t_launch) with BW, TC the measured peaks and t_launch the fastest per-launch time this
    # step measured (N = 64: the plain-graph launch floor); achieved fraction = ideal / measured
    # (this rank's points), and the effective HBM fraction over the HBM-bound points N >= 4096
    sweep_ideal = None
    rt_all = tab["runtime_ms"][:tab["n_rows"]]
    if tab["n_rows"] and np.isfinite(rt_all).any():
        t_launch = float(np.nanmin(rt_all)) * 1e-3
        ideal = meas = hb_bytes = hb_time = 0.0
        for gi, n in enumerate(SIZES):
            a, b = tab["group_offset"][gi], tab["group_offset"][gi + 1]
            if b <= a:
                continue
            nbytes_n, flops_n = L.kernel_work(L.K_EUCLID, n)
            t_pt = max(nbytes_n / (hbm_peak * 1e9), flops_n / (tc_peak * 1e12), t_launch)
            v = tab["runtime_ms"][a:b] * 1e-3
            ideal += (b - a) * (W + K * R) * t_pt
            meas += float(np.nansum(v)) * (W + K * R)
            if n >= 4096:
                hb_bytes += (b - a) * nbytes_n
                hb_time += float(np.nansum(v))
        sweep_ideal = {"t_launch_us": round(t_launch * 1e6, 3), "ideal_s": round(ideal, 3),
                       "measured_kernel_s": round(meas, 3), "achieved_fraction": round(ideal / meas, 4),
                       "hbm_frac_n_ge_4096": round(hb_bytes / hb_time / 1e9 / hbm_peak, 4) if hb_time else None,
                       "note": "per rank; warm L2 (the table's definition), so N >= 4096 can exceed 1"}
    spread = None
    if world > 1:
        objs = [None] * world
        dist.all_gather_object(objs, roof)
        roof = next((r for r in objs if r), None)
        # SURVEY 8(e) caveat: a group's blocks are timed on different GPUs; the same calibration
        # point (euclid N = 8192, block 32, 200 back-to-back launches, CUDA events) on every
        # rank gives the cross-device timing spread
        for _ in range(10):
            ctx.launch(L.K_EUCLID, 8192, 32)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        c0.record(stream)
        for _ in range(200):
            ctx.launch(L.K_EUCLID, 8192, 32)
        c1.record(stream)
        torch.cuda.synchronize()
        times = [None] * world
        dist.all_gather_object(times, c0.elapsed_time(c1) / 200 * 1e3)
        spread = {"point": "euclid N=8192 block=32, 200 stream launches", "us_by_rank": [round(x, 3) for x in times],
                  "max_over_min": round(max(times) / min(times), 4)}

    # ---- e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(ctx, L, ks, W, K, R, npts_total, world, barrier, allmax,
                      steps=min(args.steps, 2), launch_mode=launch_mode, timer=timer)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        A_by_n = {n: (ctx.suite_tensor(L.K_EUCLID, n, 0).view(n, n).cpu().numpy(),
                      ctx.suite_tensor(L.K_EUCLID, n, 1).cpu().numpy()) for n in SIZES}
        hi_ = host_info()
        v1, work1, rounds1 = oracle_points_per_s(args.policy, A_by_n, min_s=8.0)
        vn, workn, roundsn = oracle_points_per_s(args.policy, A_by_n, min_s=8.0, threads=hi_["nproc"])
        cpu = {"value": vn, "unit": "points/s", "cores": hi_["nproc"], "kind": "oracle",
               "host": hi_, "single_core_value": v1,
               "sample": f"fp64 numpy evaluations of euclidean_kernel on the same inputs (row chunks "
                         f"on {hi_['nproc']} threads; single core: {rounds1} rounds, {work1:.1f} s), "
                         f"every matrix size once per round, {roundsn} rounds ({workn:.1f} s wall), "
                         f"mean per-size time scaled by 32 blocks x (W+K*R) launches per point"}

    # ---- secondary: table rows/s (all N), the PDL launch mode, % of peak per kernel (cold L2)
    secondary = {}
    if not args.no_secondary:
        secondary["tables"] = table_benches(ctx, L, hbm_peak, rank, world, barrier, allmax,
                                            cpu_rows=(rank == 0 and world == 1 and not args.no_cpu))
        cpu_rows = secondary["tables"].pop("_cpu_rows_per_s", None)
        if cpu is not None and cpu_rows:
            cpu["table_rows_per_s"] = cpu_rows
        secondary["full_suite_fast_policy"] = full_suite_sweep(ctx, L, launch_mode, world, barrier, allmax)
        if world == 1:
            secondary["launch_modes"] = launch_mode_compare(ctx, L, ks, table, ropts, W, K, R, flush,
                                                            barrier, last[1], args.launch)
            secondary["suite_roofline_n8192"] = suite_roofline(ctx, L, hbm_peak, tc_peak)
            secondary["occupancy_api"] = occupancy_vs_sweep(ctx, L)

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 4), "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tot_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "configs[1] euclid full sweep: euclidean_kernel x blocks "
                                   "32..1024 step 32 x N 64..8192 (powers of 2)",
                       "policy": f"{args.policy}: W={W} K={K} R={R}", "points": npts_total,
                       "launch": args.launch, "timer": args.timer, "l2_table": "warm (paper)",
                       "parallelism": f"point-LPT x{world}", "l2": "flushed between steps "
                       "(512 MB write); N=8192 inputs (268 MB) exceed L2 (126 MB)"},
            "clocks": ck, "gpu_launches": launches, "roofline": roof, "roofline_warm": roof_warm,
            "cpu_baseline": cpu, "e2e": e2e, "secondary": secondary,
            "per_n_launch_us": per_n, "sweep_roofline": sweep_ideal, "cross_device_spread": spread,
            "stats_last_step": {k: last[1][k] for k in ("n_rows", "n_ratio_defined",
                                                      "n_largest_is_best", "mean_perf",
                                                      "frac_largest_not_best")},
        }
        print(json.dumps(out))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def launch_mode_compare(ctx, L, ks, table, ropts, W, K, R, flush, barrier, st_default, default):
    """The same step with the other launch mode (PDL edges between a bracket's launches: launch
    i+1 is resident while launch i drains) as a throughput secondary, with the paper's
    statistics of both tables: the runtime table depends on the launch mode."""
    import torch
    other = "graph_pdl" if default != "graph_pdl" else "graph"
    mode = {"graph": L.LAUNCH_GRAPH, "graph_pdl": L.LAUNCH_GRAPH_PDL}[other]
    flush.zero_()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = ctx.sweep(ks, SIZES, BLOCKS, warmup=W, brackets=K, launches=R, timeout_s=30.0, table=table,
                  launch_mode=mode)
    red = ctx.reduce_table(t, ropts, per_group=True)
    st = ctx.stats(ropts, percentiles=PCTS)
    e1.record()
    barrier()
    ms = e0.elapsed_time(e1)
    keys = ("n_largest_is_best", "frac_largest_not_best", "mean_perf", "mean_gain", "frac_gain_gt")
    bb = red["best_block_id"].cpu().numpy().view(np.uint16)
    return {other: {"value": round(len(SIZES) * len(BLOCKS) / (ms / 1e3), 4), "unit": "points/s",
                    "ms_per_step": round(ms, 3), "steps": 1,
                    "stats": {k: st[k] for k in keys},
                    "best_block_by_n": {str(n): BLOCKS[b] if b < len(BLOCKS) else None for n, b in zip(SIZES, bb)}},
            default: {"stats": {k: st_default[k] for k in keys}}}


def run_e2e(ctx, L, ks, W, K, R, npts_total, world, barrier, allmax, steps=2, launch_mode=0,
            timer=0):
    """Same metric through the C ABI with HOST buffers: each step uploads the suite inputs
    from pinned host memory, sweeps into a pinned host table, reduces that host table and
    reads the stats back."""
    import torch
    host_in = {}
    h2d = 0
    for n in SIZES:
        for slot in (0, 1):
            t = ctx.suite_tensor(L.K_EUCLID, n, slot).cpu().pin_memory()
            host_in[(n, slot)] = t
            h2d += t.numel() * 4
    G = len(ks) * len(SIZES)
    host_tab = L.Table.empty(npts_total, G, device="cpu", pin=True)
    ropts = L.reduce_opts(len(BLOCKS), len(SIZES), point_sharded=1 if world > 1 else 0)
    stream = torch.cuda.current_stream()

    def step():
        for (n, slot), t in host_in.items():
            ctx.suite_upload(L.K_EUCLID, n, slot, t)
        tab = ctx.sweep(ks, SIZES, BLOCKS, warmup=W, brackets=K, launches=R, table=host_tab,
                        launch_mode=launch_mode, timer=timer)
        ctx.reduce_table(tab, ropts, per_group=False)
        return ctx.stats(ropts, percentiles=PCTS), tab.n_rows

    step()
    barrier()
    ms = 0.0
    rows = 0
    for _ in range(steps):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, rows = step()
        e1.record(stream)
        barrier()
        ms += e0.elapsed_time(e1)
    ms = allmax(ms)
    plen = L.partials_len(ropts)
    tab_h2d = rows * 6 + (G + 1) * 8 + G * 4
    return {"value": round(npts_total * steps / (ms / 1e3), 4), "unit": "points/s",
            "h2d_bytes_per_step": h2d + tab_h2d, "d2h_bytes_per_step": plen * 8 + 32,
            "steps": steps, "note": "sweep runtimes come from device events read on the host; "
                                    "percentile-selection histograms not counted in d2h"}


def suite_roofline(ctx, L, hbm_peak, tc_peak, blocks=(128, 256, 512, 1024)):
    """BASELINE metric '% HBM peak per kernel': every suite kernel at N = 8192, best of a few
    blocks, per-launch time from CUDA events over 3 brackets x 20 launches with COLD L2
    (LSCAT_L2_ROTATE: >= 2 x L2 of buffer copies cycled launch by launch, no keep policies),
    so every byte counted comes from HBM."""
    names = ["euclid", "matvec", "rowsum", "colsum", "transpose", "axpy", "stencil5", "gemm_bf16"]
    ks = [L.KERNELS[k] for k in names]
    n = 8192
    ctx.register_suite(ks, [n])
    out = {}
    for name, k in zip(names, ks):
        nbytes, flops = L.kernel_work(k, n)
        t = ctx.sweep([k], [n], list(blocks), warmup=1, brackets=3, launches=20,
                      l2_mode=L.L2_ROTATE, with_brackets=True).to_numpy()
        rt = t["runtime_ms"]
        i = int(np.nanargmin(rt))
        b, ms = blocks[int(t["block_id"][i])], float(rt[i])
        if k == L.K_GEMM_BF16:
            ach = flops / (ms * 1e-3) / 1e12
            out[name] = {"bound": "tensor", "block": b, "us": round(ms * 1e3, 2),
                         "achieved": round(ach, 1), "unit": "TFLOP/s", "frac": round(ach / tc_peak, 4)}
        else:
            ach = nbytes / (ms * 1e-3) / 1e9
            out[name] = {"bound": "hbm", "block": b, "us": round(ms * 1e3, 2),
                         "achieved": round(ach, 1), "unit": "GB/s", "frac": round(ach / hbm_peak, 4)}
    out["l2"] = "cold (LSCAT_L2_ROTATE), median of 3 brackets x 20 launches, best of blocks " + str(list(blocks))
    return out


def occupancy_vs_sweep(ctx, L):
    """the block cudaOccupancyMaxPotentialBlockSize picks for each suite kernel
    (independent of N by construction) against the swept argmin per (kernel, N) of the full
    suite (fast policy), evaluated with the table reducer by taking the API's block as the
    'largest' block: its performance best / r(api) per group."""
    names = ["euclid", "matvec", "gemm_bf16", "transpose", "axpy", "rowsum", "colsum", "stencil5"]
    ks = [L.KERNELS[k] for k in names]
    ctx.register_suite(ks, SIZES)
    Wf, Kf, Rf = POLICIES["fast"]
    out = {}
    for name, k in zip(names, ks):
        api = ctx.occupancy_block(k, BLOCKS)
        sub = ctx.sweep([k], SIZES, BLOCKS, warmup=Wf, brackets=Kf, launches=Rf)
        o = L.reduce_opts(len(BLOCKS), len(SIZES), largest_block_id=api["block_id"])
        red = ctx.reduce_table(sub, o, per_group=True)
        st = ctx.stats(o)
        best = red["best_block_id"].cpu().numpy().view(np.uint16)
        perf = red["perf"].cpu().numpy()
        out[name] = {"api_block": BLOCKS[api["block_id"]], "api_min_grid": api["min_grid"],
                     "swept_best_by_n": {str(n): (BLOCKS[b] if b < len(BLOCKS) else None) for n, b in zip(SIZES, best)},
                     "api_perf_by_n": {str(n): (round(float(p), 4) if np.isfinite(p) else None) for n, p in zip(SIZES, perf)},
                     "api_is_best": st["n_largest_is_best"], "groups": st["n_ratio_defined"],
                     "mean_perf_api": round(st["mean_perf"], 4)}
    return out


def full_suite_sweep(ctx, L, launch_mode, world, barrier, allmax):
    """The whole suite (8 kernels x 32 blocks x 8 matrix sizes = 2048 points, SURVEY 8(d)
    scaling workload) swept with the fast policy (1 + 5 x 20 launches), point-LPT sharded over
    the ranks, then reduced (per-group NCCL merge when N > 1): sweep points/s (max over ranks)
    and the paper's statistics on this suite."""
    import torch
    names = ["euclid", "matvec", "gemm_bf16", "transpose", "axpy", "rowsum", "colsum", "stencil5"]
    ks = [L.KERNELS[k] for k in names]
    ctx.register_suite(ks, SIZES)
    W, K, R = POLICIES["fast"]
    o = L.reduce_opts(len(BLOCKS), len(SIZES), point_sharded=1 if world > 1 else 0)
    tab = ctx.sweep(ks, SIZES, BLOCKS, warmup=W, brackets=K, launches=R, launch_mode=launch_mode)  # warm
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tab = ctx.sweep(ks, SIZES, BLOCKS, warmup=W, brackets=K, launches=R, launch_mode=launch_mode)
    red = ctx.reduce_table(tab, o, per_group=True)
    st = ctx.stats(o, percentiles=[0.5])
    e1.record()
    barrier()
    ms = allmax(e0.elapsed_time(e1))
    bb = red["best_block_id"].cpu().numpy().view(np.uint16)
    G = len(ks) * len(SIZES)
    best = {names[gi // len(SIZES)]: BLOCKS[bb[gi]] for gi in range(G)
            if SIZES[gi % len(SIZES)] == 8192 and bb[gi] < len(BLOCKS)}
    return {"points": G * len(BLOCKS), "policy": f"fast: W={W} K={K} R={R}", "n_gpus": world,
            "points_per_s": round(G * len(BLOCKS) / (ms / 1e3), 2), "ms": round(ms, 1),
            "n_nan_rows": int(st["n_nan"]), "frac_largest_not_best": round(st["frac_largest_not_best"], 4),
            "mean_perf_largest": round(st["mean_perf"], 4), "frac_gain_gt_20pct": round(st["frac_gain_gt"], 4),
            "best_block_at_n8192": best}


TABLE_CASES = [
    ("gtx980_2140796", dict(n_rows_global=2_140_796, n_kernels=8363, preset=1, seed=980)),
    ("t4_5028536", dict(n_rows_global=5_028_536, n_kernels=19_683, preset=0, seed=4)),
    ("scaled_1e9", dict(n_rows_global=1_000_000_000, n_kernels=3_906_250, preset=0,
                        seed=10 ** 9, offsets=False)),
]


def table_benches(ctx, L, hbm_peak, rank, world, barrier, allmax, cpu_rows=False):
    """Table rows/s of reduce + merge + stats (9 percentiles) on device-resident tables,
    BASELINE configs[2]-[4] (median of 10, max over ranks).  With N ranks each rank generates
    its own shard in place: group-aligned (contiguous group ranges: only the ~11 KB partial
    vector and the percentile histograms are merged) and, for configs[2]/[3], point-sharded
    (block ids b % N == rank: the per-group MIN/MAX/SUM merge of 28 B/group first).  `local_ms`
    is the same shard reduced by a context without a communicator (no merge): the difference
    is the NCCL merge."""
    import torch
    out = {"l2": "cold: a 512 MB buffer is written before every timed rep (outside the events)"}
    cpu = {}
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    solo = L.Ctx(torch.cuda.current_device(), seed=0x15CA7) if world > 1 else None
    stream = torch.cuda.current_stream()
    for name, kw in TABLE_CASES:
        kw = dict(kw)
        offsets = kw.pop("offsets", True)
        n_glob = kw["n_rows_global"]
        shapes = [("group_aligned", False)] + ([("point_sharded", True)] if world > 1 and offsets else [])
        for shard_name, point in shapes:
            G = -(-n_glob // 32)
            if point:
                tab = ctx.gen_table(**kw, block_mod=world, block_rem=rank, offsets=offsets)
            else:
                g0, g1 = G * rank // world, G * (rank + 1) // world
                tab = ctx.gen_table(**kw, group_begin=g0, group_end=g1 if world > 1 else 0, offsets=offsets)
            # the percentiles ride in the reduce options (R-27): the selection is enqueued behind
            # the reduction and lscat_stats collects it (one rank; ignored with N > 1)
            o = L.reduce_opts(32, 8, point_sharded=1 if (point and world > 1) else 0, percentiles=PCTS)
            o2 = L.reduce_opts(32, 8, point_sharded=1 if (point and world > 1) else 0)

            def run(c, oo):
                c.reduce_table(tab, oo, per_group=False)
                return c.stats(oo, percentiles=PCTS)

            def timed(oo, reps):
                times, rtimes = [], []
                for _ in range(reps):
                    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                    flush.zero_()  # cold L2 for every timed rep (outside the events)
                    barrier()
                    e0.record(stream)
                    ctx.reduce_table(tab, oo, per_group=False)
                    e1.record(stream)
                    st_ = ctx.stats(oo, percentiles=PCTS)
                    e2.record(stream)
                    barrier()
                    times.append(allmax(e0.elapsed_time(e2)))
                    rtimes.append(allmax(e0.elapsed_time(e1)))
                return statistics.median(times), statistics.median(rtimes), st_
            for _ in range(3):
                run(ctx, o2)
            ms2, _, st2 = timed(o2, 5)  # percentiles given to lscat_stats only
            for _ in range(3):
                run(ctx, o)
            ms, rms, st = timed(o, 10)
            assert st["pct_perf"] == st2["pct_perf"] and st["pct_gain"] == st2["pct_gain"]
            key = name if world == 1 else f"{name}_{shard_name}"
            # 6 B/row read + 15 B/group of outputs + <= 0.25 B/row of refinement
            alg = tab.n_rows * 6.25 + tab.n_groups * 15
            res = {"rows_per_s": round(n_glob / (ms / 1e3), 1), "ms_reduce_plus_stats": round(ms, 4),
                   "ms_reduce_call": round(rms, 4),
                   "ms_percentiles_at_stats_only": round(ms2, 4), "n_rows_global": n_glob,
                   "rows_per_rank": tab.n_rows, "roofline_frac": round(alg / (ms * 1e-3) / 1e9 / hbm_peak, 4),
                   "check_n_rows": st["n_rows"]}
            if solo is not None:
                so = L.reduce_opts(32, 8)
                for _ in range(2):
                    run(solo, so)
                lt = []
                for _ in range(5):
                    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                    torch.cuda.synchronize()
                    e0.record(stream)
                    run(solo, so)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    lt.append(e0.elapsed_time(e1))
                res["local_ms_no_merge"] = round(allmax(statistics.median(lt)), 4)
            # the per-kernel roll-up of P:258 (R-26) on the same shard: its extra time and values
            ok_ = L.reduce_opts(32, 8, point_sharded=1 if (point and world > 1) else 0, kernel_rollup=1,
                                percentiles=PCTS)
            run(ctx, ok_)
            kt = []
            for _ in range(5):
                e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                barrier()
                e0.record(stream)
                kst = run(ctx, ok_)
                e1.record(stream)
                barrier()
                kt.append(allmax(e0.elapsed_time(e1)))
            res["with_kernel_rollup"] = {
                "ms_reduce_plus_stats": round(statistics.median(kt), 4),
                "n_kernels": kst["n_kernels"],
                "frac_kernels_largest_not_best": round(kst["frac_kernels_largest_not_best"], 4),
                "frac_kernels_perf_band": round(kst["frac_kernels_perf_band"], 5),
                "mean_kernel_perf": round(kst["mean_kernel_perf"], 5)}
            out[key] = res
            if cpu_rows and name != "scaled_1e9":
                from oracle import table as OT
                h = tab.to_numpy()
                t0 = time.perf_counter()
                OT.reduce_table(h["runtime_ms"], h["block_id"], h["group_offset"],
                                group_matrix=h["group_matrix"], percentiles=PCTS)
                one = tab.n_rows / (time.perf_counter() - t0)
                t0 = time.perf_counter()
                OT.reduce_table_parallel(h["runtime_ms"], h["block_id"], h["group_offset"],
                                         group_matrix=h["group_matrix"])
                alln = tab.n_rows / (time.perf_counter() - t0)
                cpu[name] = {"one_core": round(one, 1), "all_cores": round(alln, 1),
                             "all_cores_note": "counters + histograms (percentiles on one core)"}
            del tab
            torch.cuda.empty_cache()
    if solo is not None:
        solo.close()
    out["_cpu_rows_per_s"] = cpu
    return out


if __name__ == "__main__":
    main()
