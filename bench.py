#!/usr/bin/env python
"""Benchmark of the LS-CAT hot path on B200 (BASELINE.json metric: sweep points/s and table
rows/s; % HBM peak per kernel).

A step = one pass of the whole hot path over the configs[1] workload:
plan (a2) -> sweep `euclidean_kernel` over blocks 32..1024 step 32 x N = 64..8192 (a3-a5,
paper timing policy: 1 preheat + 10 brackets x 1000 launches, median) -> reduce the runtime
table (a6/a7, NCCL merge a9 when N > 1) -> stats with percentiles (a8/a10).
`value` = sweep points/s of the whole job (points of all ranks / max-over-ranks device time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--policy paper|fast] [--impl ours|reference]

Multi-GPU: launched by torchrun, one rank per GPU, points LPT-sharded (strong scaling: the
256-point sweep is fixed).  `--impl reference` times the CPU oracle (the tier's reference arm).
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
def oracle_points_per_s(policy, A_by_n=None, min_s=10.0):
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
            OK.euclid(A, q)
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
    ap.add_argument("--launch", choices=["graph", "graph_pdl", "stream"], default="graph_pdl",
                    help="how a bracket's launches are issued (lscat_launch_mode)")
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
    launch_mode = {"graph": L.LAUNCH_GRAPH, "graph_pdl": L.LAUNCH_GRAPH_PDL,
                   "stream": L.LAUNCH_STREAM}[args.launch]
    ks = [L.K_EUCLID]
    ctx.register_suite(ks, SIZES)
    npts_total = len(ks) * len(SIZES) * len(BLOCKS)
    my_pts = L.plan(ks, SIZES, BLOCKS, rank, world, W, K, R)
    table = L.Table.empty(npts_total, len(ks) * len(SIZES))
    ropts = L.reduce_opts(len(BLOCKS), len(SIZES), point_sharded=1 if world > 1 else 0)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        t = ctx.sweep(ks, SIZES, BLOCKS, warmup=W, brackets=K, launches=R, timeout_s=30.0,
                      table=table, with_brackets=True, launch_mode=launch_mode)
        ctx.reduce_table(t, ropts, per_group=False)
        st = ctx.stats(ropts, percentiles=PCTS)
        return t, st

    for _ in range(args.warmup):
        step()
    barrier()
    clocks = Clocks(lrank)
    l0 = ctx.launch_count()
    dev_ms = 0.0
    brackets_best = []
    last = None
    for _ in range(args.steps):
        flush.zero_()                      # L2 flushed between timed steps (outside the events)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t, st = step()
        e1.record(stream)
        barrier()
        dev_ms += e0.elapsed_time(e1)
        last = (t, st)
        brackets_best.append(t.brackets.copy())
    ck = clocks.stop()
    launches = ctx.launch_count() - l0
    tot_ms = allmax(dev_ms)
    value = npts_total * args.steps / (tot_ms / 1e3)

    # ---- roofline of the dominant kernel: euclidean_kernel at N = 8192, its best block
    tab = last[0].to_numpy()
    hbm_peak, _, peak_kind = load_peaks()
    nbytes, _ = L.kernel_work(L.K_EUCLID, 8192)
    g8 = len(SIZES) - 1
    lo, hi = tab["group_offset"][g8], tab["group_offset"][g8 + 1]
    roof = None
    if hi > lo:
        rt = tab["runtime_ms"][lo:hi]
        i = int(np.nanargmin(rt))
        best_block = BLOCKS[tab["block_id"][lo + i]]
        mean_ms = float(np.mean([b[lo + i].mean() for b in brackets_best]))
        achieved = nbytes / (mean_ms * 1e-3) / 1e9
        tr = load_traffic().get(f"euclid_8192_b{best_block}") or load_traffic().get("euclid_8192")
        all_blocks_gbs = [nbytes / (float(np.mean([b[lo + j].mean() for b in brackets_best])) * 1e-3)
                          / 1e9 for j in range(hi - lo)]
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": tr,
                "kernel": f"euclid N=8192 block={best_block}", "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": nbytes, "avg_launch_ms": round(mean_ms, 5),
                "share_of_step": round(sum(float(np.mean([b[lo + j].mean() for b in brackets_best]))
                                           for j in range(hi - lo)) * (W + K * R) / (dev_ms / args.steps), 4),
                "all_blocks_gbs_min_max": [round(min(all_blocks_gbs), 1), round(max(all_blocks_gbs), 1)]}
        # A (268 MB) is twice L2: the row kernel keeps an address-hashed fraction f of its lines
        # L2-resident across the launches of a bracket (fractional evict-last policy, share
        # 0.45 of L2); `traffic` is the DRAM bytes per launch in that steady state (committed
        # ncu capture, application replay, no cache flush), so DRAM GB/s = traffic / time
        l2 = torch.cuda.get_device_properties(lrank).L2_cache_size
        share = float(os.environ.get("LSCAT_ROW_L2FRAC", "0.45"))
        roof["l2_resident_fraction"] = round(min(1.0, share * l2 / nbytes) if share > 0 else 0.0, 4)
        if tr:
            roof["dram_gbs"] = round(tr / (mean_ms * 1e-3) / 1e9, 1)
            roof["dram_frac"] = round(tr / (mean_ms * 1e-3) / 1e9 / hbm_peak, 4)
        roof["note"] = ("frac = algorithmic bytes / time (contract); part of A is served from L2 "
                        "across the bracket's back-to-back launches, so DRAM traffic per launch "
                        "(traffic, ncu steady state) is below the algorithmic bytes and "
                        "dram_frac = traffic / time / peak is the DRAM-side fraction")
    per_n = {}
    for gi, n in enumerate(SIZES):
        a, b = tab["group_offset"][gi], tab["group_offset"][gi + 1]
        if b > a:
            v = tab["runtime_ms"][a:b] * 1e3
            per_n[str(n)] = [round(float(np.nanmin(v)), 2), round(float(np.nanmedian(v)), 2),
                             round(float(np.nanmax(v)), 2)]
            if n >= 4096:
                per_n[f"{n}_by_block"] = [round(float(x), 1) for x in v]
    rooflines = None
    spread = None
    if world > 1:
        objs = [None] * world
        dist.all_gather_object(objs, roof)
        roof = next((r for r in objs if r), None)
        # SURVEY 8(e) caveat: a group's blocks are timed on different GPUs; the same calibration
        # point (euclid N = 8192, block 32, 200 back-to-back launches, CUDA events) on every
        # rank gives the cross-device timing spread (the sweep itself shards points, so it is
        # timed here with direct launches)
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
                      steps=min(args.steps, 2), launch_mode=launch_mode)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        A_by_n = {n: (ctx.suite_tensor(L.K_EUCLID, n, 0).view(n, n).cpu().numpy(),
                      ctx.suite_tensor(L.K_EUCLID, n, 1).cpu().numpy()) for n in SIZES}
        v, work, rounds = oracle_points_per_s(args.policy, A_by_n, min_s=10.0)
        cpu = {"value": v, "unit": "points/s", "cores": 1, "kind": "oracle",
               "sample": f"fp64 numpy evaluations of euclidean_kernel on the same inputs, every "
                         f"matrix size once per round, {rounds} rounds ({work:.1f} s CPU), mean "
                         f"per-size time scaled by 32 blocks x (W+K*R) launches per point"}

    # ---- secondary: table rows/s on the paper-shaped tables, % of peak per suite kernel (N = 1)
    secondary = None
    if not args.no_secondary and world == 1:
        secondary = table_benches(ctx, L, hbm_peak)
        if args.launch == "graph_pdl":
            # the same step with plain graph brackets (no programmatic-dependent-launch edges):
            # the launch gap PDL hides, measured in the same run
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tg = ctx.sweep(ks, SIZES, BLOCKS, warmup=W, brackets=K, launches=R, timeout_s=30.0,
                           table=table, launch_mode=L.LAUNCH_GRAPH)
            ctx.reduce_table(tg, ropts, per_group=False)
            ctx.stats(ropts, percentiles=PCTS)
            e1.record(stream)
            barrier()
            gms = e0.elapsed_time(e1)
            secondary["launch_graph_no_pdl"] = {"value": round(npts_total / (gms / 1e3), 4),
                                                "unit": "points/s", "ms_per_step": round(gms, 3),
                                                "steps": 1}
        secondary["suite_roofline_n8192"] = suite_roofline(ctx, L, hbm_peak, load_peaks()[1])
        secondary["full_suite_fast_policy"] = full_suite_sweep(ctx, L, launch_mode)
        cpu_rows = secondary.pop("_cpu_rows_per_s", None)
        if cpu:
            cpu["table_rows_per_s"] = cpu_rows

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 4), "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tot_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "configs[1] euclid full sweep: euclidean_kernel x blocks "
                                   "32..1024 step 32 x N 64..8192 (powers of 2)",
                       "policy": f"{args.policy}: W={W} K={K} R={R}", "points": npts_total,
                       "launch": args.launch,
                       "parallelism": f"point-LPT x{world}", "l2": "flushed between steps "
                       "(512 MB write); N=8192 inputs (268 MB) exceed L2 (126 MB)"},
            "clocks": ck, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu,
            "e2e": e2e, "secondary": secondary,
            "per_n_launch_us": per_n, "cross_device_spread": spread,
            "stats_last_step": {k: last[1][k] for k in ("n_rows", "n_ratio_defined",
                                                      "n_largest_is_best", "mean_perf",
                                                      "frac_largest_not_best")},
        }
        print(json.dumps(out))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    del rooflines


def run_e2e(ctx, L, ks, W, K, R, npts_total, world, barrier, allmax, steps=2, launch_mode=0):
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
                        launch_mode=launch_mode)
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


def suite_roofline(ctx, L, hbm_peak, tc_peak, blocks=(128, 256, 512, 1024), reps=20):
    """BASELINE metric '% HBM peak per kernel': every suite kernel at N = 8192, best of a few
    blocks, per-launch time from CUDA events over `reps` back-to-back launches (inputs exceed
    L2 except colsum/rowsum/matvec/euclid's 256 MB, which also exceed it)."""
    import torch
    names = ["euclid", "matvec", "rowsum", "colsum", "transpose", "axpy", "stencil5", "gemm_bf16"]
    ks = [L.KERNELS[k] for k in names]
    n = 8192
    ctx.register_suite(ks, [n])
    stream = torch.cuda.current_stream()
    out = {}
    for name, k in zip(names, ks):
        nbytes, flops = L.kernel_work(k, n)
        best = None
        for b in blocks:
            ctx.launch(k, n, b)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(reps):
                ctx.launch(k, n, b)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            if best is None or ms < best[1]:
                best = (b, ms)
        b, ms = best
        if k == L.K_GEMM_BF16:
            ach = flops / (ms * 1e-3) / 1e12
            out[name] = {"bound": "tensor", "block": b, "us": round(ms * 1e3, 2),
                         "achieved": round(ach, 1), "unit": "TFLOP/s", "frac": round(ach / tc_peak, 4)}
        else:
            ach = nbytes / (ms * 1e-3) / 1e9
            out[name] = {"bound": "hbm", "block": b, "us": round(ms * 1e3, 2),
                         "achieved": round(ach, 1), "unit": "GB/s", "frac": round(ach / hbm_peak, 4)}
    return out


def full_suite_sweep(ctx, L, launch_mode):
    """The whole suite (8 kernels x 32 blocks x 8 matrix sizes = 2048 points, SURVEY 8(d)
    scaling workload) swept with the fast policy (1 + 5 x 20 launches), then reduced: sweep
    points/s and the paper's statistics on this suite."""
    import torch
    names = ["euclid", "matvec", "gemm_bf16", "transpose", "axpy", "rowsum", "colsum", "stencil5"]
    ks = [L.KERNELS[k] for k in names]
    ctx.register_suite(ks, SIZES)
    W, K, R = POLICIES["fast"]
    ctx.sweep(ks, SIZES, BLOCKS, warmup=W, brackets=K, launches=R, launch_mode=launch_mode)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tab = ctx.sweep(ks, SIZES, BLOCKS, warmup=W, brackets=K, launches=R, launch_mode=launch_mode)
    o = L.reduce_opts(len(BLOCKS), len(SIZES))
    ctx.reduce_table(tab, o, per_group=False)
    st = ctx.stats(o, percentiles=[0.5])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = tab.to_numpy()
    best = {}
    for gi in range(t["n_groups"]):
        a, b = t["group_offset"][gi], t["group_offset"][gi + 1]
        if SIZES[t["group_matrix"][gi]] != 8192 or b <= a:
            continue
        rt = t["runtime_ms"][a:b]
        if np.isfinite(rt).any():
            j = int(np.nanargmin(rt))
            best[names[ks.index(int(t["group_kernel"][gi]))]] = [BLOCKS[t["block_id"][a + j]],
                                                                  round(float(rt[j]) * 1e3, 2)]
    return {"points": int(t["n_rows"]), "policy": f"fast: W={W} K={K} R={R}",
            "points_per_s": round(t["n_rows"] / (ms / 1e3), 2), "ms": round(ms, 1),
            "n_nan_rows": int(st["n_nan"]), "frac_largest_not_best": round(st["frac_largest_not_best"], 4),
            "mean_perf_largest": round(st["mean_perf"], 4), "frac_gain_gt_20pct": round(st["frac_gain_gt"], 4),
            "best_block_us_at_n8192": best}


def table_benches(ctx, L, hbm_peak):
    """Table rows/s of reduce+stats (device-resident tables, BASELINE configs[2]-[4] at N=1)."""
    import torch
    from oracle import table as OT
    out = {}
    cpu_rows = {}
    cases = [("gtx980_2140796", dict(n_rows_global=2_140_796, n_kernels=8363, preset=L.PRESET_GTX980, seed=980)),
             ("t4_5028536", dict(n_rows_global=5_028_536, n_kernels=19_683, preset=L.PRESET_T4, seed=4)),
             ("scaled_1e9", dict(n_rows_global=1_000_000_000, n_kernels=3_906_250, preset=L.PRESET_T4,
                                 seed=10 ** 9, offsets=False))]
    stream = torch.cuda.current_stream()
    for name, kw in cases:
        tab = ctx.gen_table(**kw)
        o = L.reduce_opts(32, 8)
        for _ in range(3):
            ctx.reduce_table(tab, o, per_group=False)
            ctx.stats(o, percentiles=PCTS)
        times, rtimes = [], []
        for _ in range(10):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            torch.cuda.synchronize()
            e0.record(stream)
            ctx.reduce_table(tab, o, per_group=False)
            e1.record(stream)
            ctx.stats(o, percentiles=PCTS)
            e2.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e2))
            rtimes.append(e0.elapsed_time(e1))
        ms, rms = statistics.median(times), statistics.median(rtimes)
        G = tab.n_groups
        alg = tab.n_rows * 6 + G * 16          # runtime+block id read, perf+gain written
        out[name] = {"rows_per_s": round(tab.n_rows / (ms / 1e3), 1), "ms_reduce_plus_stats": round(ms, 4),
                     "ms_reduce_kernel_path": round(rms, 4),
                     "reduce_hbm_frac": round(alg / (rms * 1e-3) / 1e9 / hbm_peak, 4)}
        if name != "scaled_1e9":
            h = tab.to_numpy()
            t0 = time.perf_counter()
            OT.reduce_table(h["runtime_ms"], h["block_id"], h["group_offset"],
                            group_matrix=h["group_matrix"], percentiles=PCTS)
            cpu_rows[name] = round(tab.n_rows / (time.perf_counter() - t0), 1)
        del tab
        torch.cuda.empty_cache()
    out["_cpu_rows_per_s"] = cpu_rows
    return out


if __name__ == "__main__":
    main()
