"""a9 merge on one GPU: W ranks are W threads, each with its own library context, joined by the
library's local test transport (lscat_comm_init_local).  The merge code in reduce.cu /
stats.cu is the same as with NCCL; only the byte transport differs.  Every rank must get
results bit-identical to the oracle on the whole table, for point-sharded tables (per-group
MIN/MAX/SUM merge) and group-aligned shards (partial-vector SUM), for W = 2, 3, 4."""
import threading

import numpy as np
import pytest

from oracle import table as OT
from synth import gen_table
from tests.gpu_util import require_gpu

pytestmark = pytest.mark.gpu

PCTS = [0.01, 0.1, 0.5, 0.9, 0.99]


def _run_ranks(world, make_table, opts_kw, name):
    import torch
    import importlib
    importlib.import_module("paper_2103_14409_b200.build").build()
    import paper_2103_14409_b200 as L
    results, errors = [None] * world, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            ctx = L.Ctx(0)
            ctx.comm_init_local(name, r, world)
            tab = make_table(ctx, r)
            o = L.reduce_opts(32, 8, **opts_kw)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out = ctx.reduce_table(tab, o, stream=s)
                st = ctx.stats(o, percentiles=PCTS, stream=s)
            s.synchronize()
            results[r] = (st, {k: v.cpu().numpy() for k, v in out.items()})
            ctx.close()
        except Exception as e:  # noqa: BLE001
            errors.append((r, repr(e)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    return results


def _check(results, ref):
    from tests.test_gpu_reduce import _check_rollup
    for st, _ in results:
        if ref.rollup is not None:
            _check_rollup(st, ref.rollup)
        for k, v in ref.counters.items():
            assert st[k] == v, k
        assert (st["perf_hist"] == ref.perf_hist).all()
        assert (st["gain_hist"] == ref.gain_hist).all()
        assert (st["best_block_hist"] == ref.best_block_hist).all()
        assert st["pct_perf"] == ref.percentiles["perf"]
        assert st["pct_gain"] == ref.percentiles["gain"]
        assert st["mean_perf"] == ref.derived["mean_perf"]


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_point_sharded_merge(world):
    require_gpu()
    n, K = 400_000, 1601                 # 7 or 8 groups per kernel: rank ranges split kernels
    full = gen_table(n, K, preset="t4", seed=31)
    ref = OT.reduce_table(full["runtime_ms"], full["block_id"], full["group_offset"],
                          group_matrix=full["group_matrix"], percentiles=PCTS,
                          group_kernel=full["group_kernel"], kernel_rollup=True)

    def make(ctx, r):
        return ctx.gen_table(n, K, preset=0, seed=31, block_mod=world, block_rem=r)

    res = _run_ranks(world, make, dict(point_sharded=1, kernel_rollup=1), f"ps{world}")
    _check(res, ref)
    # every rank holds the merged per-group argmin for all groups
    for _, out in res:
        assert (out["best_block_id"].view(np.uint16) == ref.best_block).all()


def test_point_sharded_host_tables():
    """The e2e leg of bench.py at N > 1: every rank reduces a pinned HOST table of its own
    points (staged through device scratch by the library) with the point-sharded merge; the
    merged statistics equal the whole-table oracle (local transport, 2 ranks)."""
    require_gpu()
    import torch
    from paper_2103_14409_b200 import MEM_HOST
    n, K = 300_000, 1201
    full = gen_table(n, K, preset="t4", seed=37)
    ref = OT.reduce_table(full["runtime_ms"], full["block_id"], full["group_offset"],
                          group_matrix=full["group_matrix"], percentiles=PCTS)

    def make(ctx, r):
        d = ctx.gen_table(n, K, preset=0, seed=37, block_mod=2, block_rem=r)
        for k in ("runtime_ms", "block_id", "status", "group_offset", "group_kernel", "group_matrix"):
            v = getattr(d, k)
            if v is not None:
                setattr(d, k, v.cpu().pin_memory())
        torch.cuda.synchronize()
        d.mem = MEM_HOST
        return d

    res = _run_ranks(2, make, dict(point_sharded=1), "psh2")
    _check(res, ref)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_group_aligned_merge(world):
    require_gpu()
    n, K = 32 * 120_000, 15_001
    full = gen_table(n, K, preset="gtx980", seed=41)
    ref = OT.reduce_table(full["runtime_ms"], full["block_id"], full["group_offset"],
                          group_matrix=full["group_matrix"], percentiles=PCTS,
                          group_kernel=full["group_kernel"], kernel_rollup=True)
    G = full["n_groups"]

    def make(ctx, r):
        return ctx.gen_table(n, K, preset=1, seed=41, group_begin=G * r // world,
                             group_end=G * (r + 1) // world)

    res = _run_ranks(world, make, dict(kernel_rollup=1), f"ga{world}")
    _check(res, ref)


@pytest.mark.parametrize("world,point", [(2, True), (3, False)])
def test_sampled_selection_multirank(world, point):
    """The sampled first level of the percentile selection (> 2^20 keys per rank) over the local
    transport: sample histograms and interval counts summed over ranks, copies per rank."""
    require_gpu()
    n, K = 36 * 2 ** 21 if point else 3 * 36 * 2 ** 20, 300_000
    full = gen_table(n, K, preset="t4", seed=91)
    ref = OT.reduce_table(full["runtime_ms"], full["block_id"], full["group_offset"],
                          group_matrix=full["group_matrix"], percentiles=PCTS)
    G = full["n_groups"]

    def make(ctx, r):
        if point:
            return ctx.gen_table(n, K, preset=0, seed=91, block_mod=world, block_rem=r)
        return ctx.gen_table(n, K, preset=0, seed=91, group_begin=G * r // world,
                             group_end=G * (r + 1) // world)

    res = _run_ranks(world, make, dict(point_sharded=1) if point else {}, f"smp{world}{int(point)}")
    _check(res, ref)


@pytest.mark.parametrize("world", [2, 3])
def test_point_sharded_sweep_then_reduce(world):
    """a2 -> a9 end to end at world > 1 (local transport, ranks = threads on one GPU): every rank
    sweeps the points the LPT plan gives it, reduces its point-sharded table with the per-group
    merge, and every rank's statistics equal the oracle on the union of the ranks' rows."""
    require_gpu()
    import torch
    import importlib
    importlib.import_module("paper_2103_14409_b200.build").build()
    import paper_2103_14409_b200 as L
    ks = [L.K_EUCLID, L.K_MATVEC, L.K_AXPY]
    ns = [64, 128, 256]
    bs = [32, 64, 128, 256, 512, 1024]
    results, tables, errors = [None] * world, [None] * world, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            ctx = L.Ctx(0)
            ctx.comm_init_local(f"sw{world}", r, world)
            ctx.register_suite(ks, ns)
            tab = ctx.sweep(ks, ns, bs, warmup=1, brackets=3, launches=10)
            tables[r] = tab.to_numpy()
            o = L.reduce_opts(len(bs), len(ns), point_sharded=1)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx.reduce_table(tab, o, per_group=False, stream=s)
                st = ctx.stats(o, percentiles=PCTS, stream=s)
            s.synchronize()
            results[r] = st
            ctx.close()
        except Exception as e:  # noqa: BLE001
            errors.append((r, repr(e)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    # the union table: every group's rows from all ranks, block ids ascending
    G = len(ks) * len(ns)
    assert sum(t["n_rows"] for t in tables) == G * len(bs)
    rt, bid, off = [], [], [0]
    for g in range(G):
        rows = []
        for t in tables:
            a, b = t["group_offset"][g], t["group_offset"][g + 1]
            rows += list(zip(t["block_id"][a:b], t["runtime_ms"][a:b]))
        rows.sort()
        assert [x[0] for x in rows] == list(range(len(bs)))      # every point swept exactly once
        bid += [x[0] for x in rows]
        rt += [x[1] for x in rows]
        off.append(len(rt))
    gm = np.tile(np.arange(len(ns), dtype=np.uint32), len(ks))
    ref = OT.reduce_table(np.array(rt, np.float32), np.array(bid, np.uint16), np.array(off, np.int64),
                          group_matrix=gm, opts=OT.Opts(n_blocks=len(bs), n_matrices=len(ns)),
                          percentiles=PCTS)
    for st in results:
        for k, v in ref.counters.items():
            assert st[k] == v, k
        assert (st["best_block_hist"] == ref.best_block_hist).all()
        assert st["pct_perf"] == ref.percentiles["perf"] and st["pct_gain"] == ref.percentiles["gain"]


@pytest.mark.parametrize("world", [1, 2, 3])
def test_implicit_kernel_rollup_shards(world):
    """The per-kernel roll-up with implicit kernel ids (no group_kernel array: kernel =
    (first_group + g) / 8, configs[4]'s layout) runs the aligned-chunk roll-up kernel;
    group-aligned shards whose boundaries cut kernels hand those kernels to the boundary merge.
    Roll-up values bit-exact against the oracle on the whole table."""
    require_gpu()
    K = 20_003                          # G / 2, G / 3 not multiples of 8: shards cut kernels
    n = 32 * 8 * K                      # G = 8 K: every kernel has exactly 8 groups
    full = gen_table(n, K, preset="t4", seed=77)
    G = full["n_groups"]
    ref = OT.reduce_table(full["runtime_ms"], full["block_id"], full["group_offset"],
                          group_matrix=full["group_matrix"], percentiles=PCTS,
                          group_kernel=np.arange(G, dtype=np.uint32) // 8, kernel_rollup=True)

    def make(ctx, r):
        return ctx.gen_table(n, K, preset=0, seed=77, group_begin=G * r // world,
                             group_end=G * (r + 1) // world if world > 1 else 0, offsets=False)

    res = _run_ranks(world, make, dict(kernel_rollup=1), f"ir{world}")
    _check(res, ref)
