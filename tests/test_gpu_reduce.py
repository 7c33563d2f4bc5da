"""a6-a10 parity: the CUDA table reducer against the C oracle on identical tables.

Integer outputs (argmin block ids, every counter, every histogram bin, fixed-point sums) and
the selected percentile values must be bit-exact; per-group perf/gain doubles too (one IEEE
division each).  Tables: the generator's GTX 980- and T4-scale tables
(BASELINE configs[2], [3]), ragged / point-sharded shapes, random tables with ties, NaN,
inf, zero and negative runtimes."""
import numpy as np
import pytest

from oracle import table as OT
from synth import gen_table
from tests.gpu_util import ctx
from tests.test_oracle_table import _random_table

pytestmark = pytest.mark.gpu

PCTS = [0.0, 0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99, 1.0]


def _device_table(t, host=False):
    import torch
    from paper_2103_14409_b200 import Table, MEM_HOST
    dev = "cpu" if host else "cuda"
    kw = dict(pin_memory=True) if host else dict(device=dev)

    def T(a, dt):
        x = torch.from_numpy(np.ascontiguousarray(a).view(dt))
        return x.pin_memory() if host else x.to(dev)
    tab = Table(T(t["runtime_ms"], np.float32), T(t["block_id"].astype(np.uint16), np.int16),
                None, T(t["group_offset"].astype(np.int64), np.int64),
                T(t["group_kernel"].astype(np.uint32), np.int32) if t.get("group_kernel") is not None else None,
                T(t["group_matrix"].astype(np.uint32), np.int32) if t.get("group_matrix") is not None else None,
                n_rows=len(t["runtime_ms"]), n_groups=len(t["group_offset"]) - 1,
                first_group=t.get("first_group", 0))
    if host:
        tab.mem = MEM_HOST
    del kw
    return tab


def _opts_pair(L=32, M=8, ell=None, policy=0, rollup=0, early=None):
    from paper_2103_14409_b200 import reduce_opts
    ell = L - 1 if ell is None else ell
    kw = dict(percentiles=early) if early is not None else {}
    g = reduce_opts(L, M, largest_block_id=ell, nan_policy=policy, kernel_rollup=rollup, **kw)
    o = OT.Opts(n_blocks=L, largest_block_id=ell, n_matrices=M, nan_policy=policy)
    return g, o


def _check_rollup(st, R):
    """Per-kernel roll-up (R-26) against the oracle: counters, histogram, fractions, mean."""
    for k_gpu, k_or in (("n_kernels", "n_kernels"), ("n_kernels_largest_not_best", "n_kernels_not_best"),
                        ("n_kernels_perf_lt", "n_kernels_perf_lt"), ("n_kernels_perf_band", "n_kernels_perf_band"),
                        ("kernel_mean_fx_hi", "kernel_mean_fx_hi"), ("kernel_mean_fx_lo", "kernel_mean_fx_lo")):
        assert st[k_gpu] == R[k_or], (k_gpu, st[k_gpu], R[k_or])
    assert (st["kernel_perf_hist"] == R["perf_hist"]).all()
    assert st["frac_kernels_largest_not_best"] == R["frac_kernels_not_best"] or R["n_kernels"] == 0
    assert st["frac_kernels_perf_band"] == R["frac_kernels_perf_band"] or R["n_kernels"] == 0


def _compare(t, L=32, M=8, ell=None, policy=0, host=False, pcts=PCTS, rollup=0, early=False):
    """early: the percentiles ride in the reduce options (R-27: selected while reducing)."""
    c = ctx()
    g_opts, o_opts = _opts_pair(L, M, ell, policy, rollup, early=pcts if early else None)
    tab = _device_table(t, host=host)
    out = c.reduce_table(tab, g_opts)
    st = c.stats(g_opts, percentiles=pcts)
    ref = OT.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                          group_matrix=t.get("group_matrix"), first_group=t.get("first_group", 0),
                          opts=o_opts, percentiles=pcts, group_kernel=t.get("group_kernel"),
                          kernel_rollup=bool(rollup))
    if rollup:
        _check_rollup(st, ref.rollup)
    for k, v in ref.counters.items():
        assert st[k] == v, (k, st[k], v)
    assert (st["perf_hist"] == ref.perf_hist).all()
    assert (st["gain_hist"] == ref.gain_hist).all()
    assert (st["best_block_hist"] == ref.best_block_hist).all()
    for k, v in ref.derived.items():
        assert (st[k] == v) or (np.isnan(st[k]) and np.isnan(v)), k
    bb = out["best_block_id"].cpu().numpy().view(np.uint16)
    assert (bb == ref.best_block).all()
    br = out["best_runtime"].cpu().numpy()
    assert (br.view(np.uint32) == ref.best_runtime.view(np.uint32)).all()
    pf = out["perf"].cpu().numpy()
    gn = out["gain"].cpu().numpy()
    assert ((pf == ref.perf) | (np.isnan(pf) & np.isnan(ref.perf))).all()
    assert ((gn == ref.gain) | (np.isnan(gn) & np.isnan(ref.gain))).all()
    assert (out["flags"].cpu().numpy().view(np.uint32) == ref.flags).all()
    if st["n_ratio_defined"]:
        assert st["pct_perf"] == ref.percentiles["perf"]
        assert st["pct_gain"] == ref.percentiles["gain"]
    return st


def test_gtx980_scale_table():
    """BASELINE configs[2]: 2 140 796 rows, ~3 % NaN."""
    t = gen_table(2_140_796, 8363, preset="gtx980", nan_rate=0.03, seed=980)
    st = _compare(t, rollup=1)
    assert st["n_rows"] == 2_140_796 and st["n_groups"] == 66_900


@pytest.mark.parametrize("policy", [0, 1])
def test_t4_scale_table(policy):
    """BASELINE configs[3]: 5 028 536 runtimes over 19 683 kernel ids."""
    t = gen_table(5_028_536, 19_683, preset="t4", nan_rate=0.03, seed=4)
    _compare(t, policy=policy, rollup=1)


def test_point_sharded_shape_and_host_table():
    t = gen_table(200_000, 800, preset="t4", nan_rate=0.05, seed=5, block_mod=3, block_rem=1)
    _compare(t)
    _compare(t, host=True, rollup=1)


@pytest.mark.parametrize("seed", range(4))
def test_random_tables_with_ties_and_invalid(seed):
    rng = np.random.default_rng(100 + seed)
    L = [4, 8, 32, 40][seed]
    rt, bid, off, gm = _random_table(rng, 3000, L, dup_vals=seed % 2 == 0)
    t = dict(runtime_ms=rt, block_id=bid, group_offset=off, group_matrix=gm)
    _compare(t, L=L, ell=L // 2 if seed == 1 else None)


def test_scale_invariance_on_gpu():
    t = gen_table(100_000, 400, preset="gtx980", seed=9)
    a = _compare(t)
    t2 = dict(t, runtime_ms=(t["runtime_ms"] * np.float32(8.0)).astype(np.float32))
    b = _compare(t2)
    for k in ("n_ratio_defined", "n_gain_gt", "perf_fx_hi", "perf_fx_lo", "pct_perf"):
        assert a[k] == b[k]


def test_generator_twin_bit_exact():
    """lscat_gen_table (CUDA) reproduces synth/tables.py bit for bit."""
    c = ctx()
    for kw in (dict(n_rows_global=2_140_796, n_kernels=8363, preset=1, seed=980),
               dict(n_rows_global=5_028_536, n_kernels=19_683, preset=0, seed=4,
                    block_mod=4, block_rem=3),
               dict(n_rows_global=1_000_000, n_kernels=100, preset=0, seed=7, group_begin=5000,
                    group_end=20000)):
        g = c.gen_table(**kw).to_numpy()
        pkw = dict(kw)
        n, k = pkw.pop("n_rows_global"), pkw.pop("n_kernels")
        pkw["preset"] = pkw["preset"]
        h = gen_table(n, k, **pkw)
        assert g["n_rows"] == h["n_rows"]
        assert (g["runtime_ms"].view(np.uint32) == h["runtime_ms"].view(np.uint32)).all()
        assert (g["block_id"] == h["block_id"]).all()
        assert (g["status"] == h["status"]).all()
        assert (g["group_offset"] == h["group_offset"]).all()
        assert (g["group_kernel"] == h["group_kernel"]).all()
        assert (g["group_matrix"] == h["group_matrix"]).all()


def test_uniform_groups_without_offsets():
    """configs[4] layout: uniform 32-row groups, no offset array, matrix = g mod 8."""
    c = ctx()
    from paper_2103_14409_b200 import reduce_opts
    n = 32 * 50_000
    tab = c.gen_table(n, 6250, preset=0, seed=10 ** 9, offsets=False)
    assert tab.rows_per_group == 32
    o = reduce_opts(32, 8)
    c.reduce_table(tab, o, per_group=False)
    st = c.stats(o, percentiles=PCTS)
    h = gen_table(n, 6250, preset="t4", seed=10 ** 9)
    ref = OT.reduce_table(h["runtime_ms"], h["block_id"], rows_per_group=32, opts=OT.Opts(),
                          percentiles=PCTS)
    for k, v in ref.counters.items():
        assert st[k] == v, k
    assert (st["best_block_hist"] == ref.best_block_hist).all()
    assert st["pct_perf"] == ref.percentiles["perf"]


def test_degenerate_tables():
    """Empty groups, an all-NaN table, a single row, a zero-group table."""
    c = ctx()
    from paper_2103_14409_b200 import reduce_opts
    # groups with 0 rows between regular ones
    t = dict(runtime_ms=np.array([1.0, 2.0, np.nan, 3.0], np.float32),
             block_id=np.array([0, 1, 0, 3], np.uint16),
             group_offset=np.array([0, 0, 2, 2, 3, 4, 4], np.int64),
             group_matrix=np.array([0, 1, 2, 3, 0, 1], np.uint32))
    st = _compare(t, L=4, M=4)
    assert st["n_groups"] == 6 and st["n_all_nan"] == 4
    # all NaN
    t = dict(runtime_ms=np.full(64, np.nan, np.float32), block_id=np.tile(np.arange(32), 2).astype(np.uint16),
             group_offset=np.array([0, 32, 64], np.int64), group_matrix=np.array([0, 1], np.uint32))
    st = _compare(t)
    assert st["n_ratio_defined"] == 0 and np.isnan(st["mean_perf"])
    assert all(np.isnan(v) for v in st["pct_perf"])
    # one row, the largest block
    t = dict(runtime_ms=np.array([0.5], np.float32), block_id=np.array([31], np.uint16),
             group_offset=np.array([0, 1], np.int64), group_matrix=np.array([5], np.uint32))
    st = _compare(t)
    assert st["n_largest_is_best"] == 1 and st["pct_perf"][0] == 1.0
    # zero groups
    import torch
    from paper_2103_14409_b200 import Table
    tab = Table(torch.zeros(1, device="cuda"), torch.zeros(1, dtype=torch.int16, device="cuda"), None,
                torch.zeros(1, dtype=torch.int64, device="cuda"), None, None, n_rows=0, n_groups=0)
    o = reduce_opts(32, 8)
    c.reduce_table(tab, o, per_group=False)
    st = c.stats(o, percentiles=[0.5])
    assert st["n_groups"] == 0 and st["n_rows"] == 0 and np.isnan(st["pct_perf"][0])


def test_group_aligned_shard_without_matrix_array():
    """A group-aligned shard (first_group != 0) with implicit matrix = (first_group + g) % M."""
    c = ctx()
    from paper_2103_14409_b200 import reduce_opts
    n = 32 * 40_000
    g0, g1 = 12_345, 30_000
    tab = c.gen_table(n, 5000, preset=0, seed=77, group_begin=g0, group_end=g1, offsets=False)
    assert tab.first_group == g0 and tab.rows_per_group == 32
    o = reduce_opts(32, 8)
    c.reduce_table(tab, o, per_group=False)
    st = c.stats(o, percentiles=PCTS)
    h = gen_table(n, 5000, preset="t4", seed=77, group_begin=g0, group_end=g1)
    ref = OT.reduce_table(h["runtime_ms"], h["block_id"], rows_per_group=32, first_group=g0,
                          opts=OT.Opts(), percentiles=PCTS)
    for k, v in ref.counters.items():
        assert st[k] == v, k
    assert (st["best_block_hist"] == ref.best_block_hist).all()
    assert st["pct_gain"] == ref.percentiles["gain"]


@pytest.mark.parametrize("policy", [0, 1])
def test_block_profile(policy):
    """Figs. 2/4 block profile (R-22): per (matrix, block) sums of floor(RN(best/r_b) 2^31) and
    counts, bit-exact vs the oracle, on a ragged table and on a uniform one."""
    c = ctx()
    from paper_2103_14409_b200 import reduce_opts
    t = gen_table(300_000, 1200, preset="t4", nan_rate=0.05, seed=12, block_mod=2, block_rem=0)
    o = reduce_opts(32, 8, nan_policy=policy, block_profile=1)
    c.reduce_table(_device_table(t), o, per_group=False)
    st = c.stats(o)
    ref = OT.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                          group_matrix=t["group_matrix"],
                          opts=OT.Opts(nan_policy=policy, block_profile=True))
    assert (st["profile_count"] == ref.profile_count).all()
    m = ~np.isnan(ref.profile_mean)
    assert (st["profile_mean"][m] == ref.profile_mean[m]).all()
    assert np.isnan(st["profile_mean"][~m]).all()
    for k, v in ref.counters.items():
        assert st[k] == v, k
    # uniform 32-row layout (vector reducer path)
    n = 32 * 30_000
    tab = c.gen_table(n, 3750, preset=0, seed=99, offsets=False)
    c.reduce_table(tab, o, per_group=False)
    st = c.stats(o)
    h = gen_table(n, 3750, preset="t4", seed=99)
    ref = OT.reduce_table(h["runtime_ms"], h["block_id"], rows_per_group=32,
                          opts=OT.Opts(nan_policy=policy, block_profile=True))
    assert (st["profile_count"] == ref.profile_count).all()
    assert (st["profile_mean"] == ref.profile_mean).all()


@pytest.mark.parametrize("ell", [31, 7])
def test_uniform_groups_unsorted_rows(ell):
    """Uniform 32-row groups whose rows are NOT in block order (the vector reducer's
    general second pass), with NaN/inf/zero rows, vs the oracle."""
    import torch
    from paper_2103_14409_b200 import Table, reduce_opts
    c = ctx()
    rng = np.random.default_rng(ell)
    h = gen_table(32 * 20_000, 2500, preset="t4", seed=21, nan_rate=0.05)
    rt, bid = h["runtime_ms"].copy(), h["block_id"].copy()
    G = h["n_groups"]
    perm = np.argsort(rng.random((G, 32)), axis=1) + (np.arange(G) * 32)[:, None]
    sel = rng.random(G) < 0.5                      # half the groups permuted, half sorted
    idx = np.where(sel[:, None], perm, (np.arange(G) * 32)[:, None] + np.arange(32)).ravel()
    rt, bid = rt[idx], bid[idx]
    bad = rng.random(rt.size) < 0.01
    rt[bad] = rng.choice(np.array([np.inf, 0.0, -1.0], np.float32), size=int(bad.sum()))
    tab = Table(torch.from_numpy(rt).cuda(), torch.from_numpy(bid.view(np.int16)).cuda(), None, None,
                None, None, n_rows=rt.size, n_groups=G, rows_per_group=32)
    o = reduce_opts(32, 8, largest_block_id=ell)
    out = c.reduce_table(tab, o)
    st = c.stats(o, percentiles=PCTS)
    ref = OT.reduce_table(rt, bid, rows_per_group=32, opts=OT.Opts(largest_block_id=ell),
                          percentiles=PCTS)
    for k, v in ref.counters.items():
        assert st[k] == v, k
    assert (out["best_block_id"].cpu().numpy().view(np.uint16) == ref.best_block).all()
    assert (out["flags"].cpu().numpy().view(np.uint32) == ref.flags).all()
    assert st["pct_perf"] == ref.percentiles["perf"]


def test_percentiles_wide_key_span_many_targets():
    """a8 with 64 percentiles over perf/gain spanning > 200 binades (gain from 2^-23 to 1e60,
    perf down to 1e-60), exact ties at perf == 1 / gain == 0: exercises the level-0 range whose
    low binades share one bin, multi-level refinement and many targets per range."""
    rng = np.random.default_rng(7)
    G = 200_000
    b = rng.uniform(0.5, 2.0, G).astype(np.float32)
    kind = rng.integers(0, 5, G)
    b = np.where(kind == 1, np.float32(1e-30), b).astype(np.float32)
    t = np.where(kind == 0, np.nextafter(b, np.float32(np.inf)),
                 np.where(kind == 1, np.float32(1e30),
                          np.where(kind == 2, b, b * rng.uniform(1.0, 3.0, G).astype(np.float32))))
    rt = np.empty(2 * G, np.float32)
    rt[0::2], rt[1::2] = b, t.astype(np.float32)
    tab = dict(runtime_ms=rt, block_id=np.tile(np.array([0, 1], np.uint16), G),
               group_offset=np.arange(0, 2 * G + 1, 2, dtype=np.int64),
               group_matrix=np.zeros(G, np.uint32))
    st = _compare(tab, L=2, M=1, ell=1, pcts=list(np.linspace(0.0, 1.0, 64)))
    assert st["pct_gain"][-1] > 1e59 and st["pct_perf"][0] < 1e-59


@pytest.mark.parametrize("early", [False, True])
def test_small_selection_ties_and_wide_bins(early):
    """The one-launch small-table selection (<= 2^20 groups) where the targets' level-0 bins hold
    thousands of keys with heavy ties (40 % of the groups take one of 50 perf values, ~2400
    groups each, a few values per bin) and the bins span ~2^40 key units (perf over ~1.6
    binades): the per-bin radix select runs several 8-bit digits with long runs of equal keys;
    also bins of 129-1000 keys and the rank-counting path below 128.  Exact against the oracle,
    with the percentiles given to lscat_stats and in the reduce options (R-27)."""
    rng = np.random.default_rng(23)
    G = 300_000
    b = rng.choice(np.array([0.5, 1.0, 2.0, 4.0], np.float32), G)   # powers of two: b / (b tv) == 1 / tv
    tied = rng.random(G) < 0.4
    tv = np.where(tied, rng.choice(np.linspace(1.05, 1.2, 50).astype(np.float32), G),
                  rng.uniform(1.0, 3.0, G).astype(np.float32)).astype(np.float32)
    rt = np.empty(2 * G, np.float32)
    rt[0::2], rt[1::2] = b, (b * tv).astype(np.float32)
    tab = dict(runtime_ms=rt, block_id=np.tile(np.array([0, 1], np.uint16), G),
               group_offset=np.arange(0, 2 * G + 1, 2, dtype=np.int64),
               group_matrix=np.zeros(G, np.uint32))
    pcts = [0.001, 0.01, 0.05, 0.1, 0.2, 0.25, 0.3, 0.35, 0.4, 0.5, 0.6, 0.75, 0.9, 0.99, 0.999, 1.0]
    _compare(tab, L=2, M=1, ell=1, pcts=pcts, early=early)


def test_percentiles_dense_bin_compaction():
    """a8 where one level-0 bin holds ~35 % of the ratio-defined groups as distinct keys
    (perf = 1 - j * 2^-20): the level-1 range is too large to gather, so the device copies the
    keys of the open ranges out and refines on the copies (percentile select)."""
    rng = np.random.default_rng(11)
    G = 400_000
    b = rng.uniform(0.5, 2.0, G).astype(np.float32)
    dense = rng.random(G) < 0.35
    j = rng.integers(1, 1 << 8, G).astype(np.float32)
    t = np.where(dense, b * (np.float32(1) + j * np.float32(2.0 ** -20)),
                 b * rng.uniform(1.0, 4.0, G).astype(np.float32)).astype(np.float32)
    rt = np.empty(2 * G, np.float32)
    rt[0::2], rt[1::2] = b, t
    tab = dict(runtime_ms=rt, block_id=np.tile(np.array([0, 1], np.uint16), G),
               group_offset=np.arange(0, 2 * G + 1, 2, dtype=np.int64),
               group_matrix=np.zeros(G, np.uint32))
    _compare(tab, L=2, M=1, ell=1, pcts=[0.01, 0.2, 0.5, 0.7, 0.8, 0.9, 0.95, 0.99])


def test_scaled_table_1e9_sampled():
    """configs[4] at full size, the configuration bench.py times: 10^9 rows = 31.25 M uniform
    32-row groups (no offset array).  Whole-table oracle comparison at the end.  The counters obey every invariant; per-group outputs are
    bit-exact against the oracle on sampled windows of groups (their rows regenerated by the
    CPU twin of the generator and compared byte for byte first); every percentile satisfies the
    nearest-rank property over the device's per-group values (properties that hold at any
    size, R-13)."""
    import torch
    from paper_2103_14409_b200 import reduce_opts, PRESET_T4
    c = ctx()
    n, K, L, M = 1_000_000_000, 3_906_250, 32, 8
    G = n // L
    tab = c.gen_table(n, K, preset=PRESET_T4, seed=10 ** 9, offsets=False)
    o = reduce_opts(L, M, kernel_rollup=1)
    out = c.reduce_table(tab, o)
    st = c.stats(o, percentiles=PCTS)
    assert st["n_rows"] == n and st["n_groups"] == G
    assert st["n_ok"] + st["n_nan"] + st["n_invalid"] == n
    nrd = st["n_ratio_defined"]
    assert int(st["perf_hist"].sum()) == nrd == int(st["gain_hist"].sum())
    assert int(st["best_block_hist"].sum()) == st["n_defined"]
    assert st["n_largest_is_best"] <= nrd and st["n_gain_gt"] <= nrd
    # sampled windows of 256 groups (first, last and six inside) vs the oracle
    W = 256
    rng = np.random.default_rng(1)
    starts = [0, G - W] + sorted(int(x) for x in rng.integers(1, G - W, 6))
    for g0 in starts:
        h = gen_table(n, K, preset="t4", seed=10 ** 9, group_begin=g0, group_end=g0 + W)
        r0, r1 = g0 * L, (g0 + W) * L
        dev_rt = tab.runtime_ms[r0:r1].cpu().numpy()
        dev_id = tab.block_id[r0:r1].cpu().numpy().view(np.uint16)
        assert (dev_rt.view(np.uint32) == h["runtime_ms"].view(np.uint32)).all()
        assert (dev_id == h["block_id"]).all()
        ref = OT.reduce_table(h["runtime_ms"], h["block_id"], rows_per_group=L, first_group=g0,
                              opts=OT.Opts(n_blocks=L, n_matrices=M))
        sl = slice(g0, g0 + W)
        assert (out["best_block_id"][sl].cpu().numpy().view(np.uint16) == ref.best_block).all()
        assert (out["best_runtime"][sl].cpu().numpy().view(np.uint32) == ref.best_runtime.view(np.uint32)).all()
        pf, gn = out["perf"][sl].cpu().numpy(), out["gain"][sl].cpu().numpy()
        assert ((pf == ref.perf) | (np.isnan(pf) & np.isnan(ref.perf))).all()
        assert ((gn == ref.gain) | (np.isnan(gn) & np.isnan(ref.gain))).all()
        assert (out["flags"][sl].cpu().numpy().view(np.uint32) == ref.flags).all()
    # nearest rank: the k-th smallest value v (k = clamp(ceil(p n), 1, n)) has fewer than k
    # values below it and at least k at or below it
    for q, vals in (("perf", st["pct_perf"]), ("gain", st["pct_gain"])):
        x = out[q]
        for p, v in zip(PCTS, vals):
            k = min(max(int(np.ceil(p * nrd)), 1), nrd)
            lt = int((x < v).sum().item())
            le = int((x <= v).sum().item())
            assert lt < k <= le, (q, p, v, lt, k, le)
    # the whole table through the oracle: group-aligned chunks of the device table
    # (the generator twin, bit-exact with synth.gen_table as checked above and in
    # test_generator_twin_bit_exact) reduced by the C oracle; every counter and histogram is a
    # sum of integer partials, so the chunked totals equal the whole-table values exactly.  The
    # percentiles are the nearest-rank values of the concatenated oracle per-group values.
    CH = 3_906_256                     # a multiple of M: chunks hold whole kernels (g // 8)
    tot = {k: 0 for k in OT.COUNTERS}
    rtot = {k: 0 for k in OT.ROLLUP}
    rh = np.zeros(101, np.uint64)
    ph = np.zeros(101, np.uint64)
    gh = np.zeros(1001, np.uint64)
    bh = np.zeros((M, L), np.uint64)
    perfs, gains = [], []
    for g0 in range(0, G, CH):
        g1 = min(G, g0 + CH)
        rt = tab.runtime_ms[g0 * L:g1 * L].cpu().numpy()
        bid = tab.block_id[g0 * L:g1 * L].cpu().numpy().view(np.uint16)
        ref = OT.reduce_table(rt, bid, rows_per_group=L, first_group=g0,
                              opts=OT.Opts(n_blocks=L, n_matrices=M), kernel_rollup=True)
        for k, v in ref.counters.items():
            tot[k] += v
        for k in OT.ROLLUP:
            rtot[k] += ref.rollup[k]
        rh += ref.rollup["perf_hist"]
        ph += ref.perf_hist
        gh += ref.gain_hist
        bh += ref.best_block_hist
        rd = (ref.flags & 0x008) != 0
        perfs.append(ref.perf[rd])
        gains.append(ref.gain[rd])
        del rt, bid, ref
    for k, v in tot.items():
        assert st[k] == v, (k, st[k], v)
    assert (st["perf_hist"] == ph).all() and (st["gain_hist"] == gh).all()
    assert (st["best_block_hist"] == bh).all()
    rtot["perf_hist"] = rh
    nk = rtot["n_kernels"]
    rtot["frac_kernels_not_best"] = rtot["n_kernels_not_best"] / nk
    rtot["frac_kernels_perf_band"] = rtot["n_kernels_perf_band"] / nk
    _check_rollup(st, rtot)
    for q, vals, parts in (("perf", st["pct_perf"], perfs), ("gain", st["pct_gain"], gains)):
        allv = np.sort(np.concatenate(parts))
        assert allv.size == nrd
        for p, v in zip(PCTS, vals):
            k = min(max(int(np.ceil(p * nrd)), 1), nrd)
            assert v == allv[k - 1], (q, p, v, allv[k - 1])
    del out, tab
    torch.cuda.empty_cache()


def _uniform_device_table(rt, bid):
    import torch
    from paper_2103_14409_b200 import Table
    n = rt.size
    return Table(torch.from_numpy(rt).cuda(), torch.from_numpy(bid.view(np.int16)).cuda(), None,
                 None, None, None, n_rows=n, n_groups=-(-n // 32), rows_per_group=32)


@pytest.mark.parametrize("n_groups,short", [(64, 5), (96, 31), (33, 1), (32, 0)])
def test_uniform_short_last_group(n_groups, short):
    """a short last group inside what would be a full 32-group batch of the uniform
    32-row path (n_groups % 32 == 0, n_rows % 32 != 0) must be bounded by n_rows."""
    c = ctx()
    from paper_2103_14409_b200 import reduce_opts
    rng = np.random.default_rng(n_groups + short)
    n = 32 * n_groups - short
    rt = rng.uniform(0.5, 2.0, n).astype(np.float32)
    rt[rng.random(n) < 0.05] = np.nan
    bid = np.tile(np.arange(32, dtype=np.uint16), n_groups)[:n].copy()
    tab = _uniform_device_table(rt, bid)
    o = reduce_opts(32, 8)
    c.reduce_table(tab, o, per_group=False)
    st = c.stats(o, percentiles=PCTS)
    ref = OT.reduce_table(rt, bid, rows_per_group=32, opts=OT.Opts(), percentiles=PCTS)
    for k, v in ref.counters.items():
        assert st[k] == v, (k, st[k], v)
    assert (st["perf_hist"] == ref.perf_hist).all() and (st["gain_hist"] == ref.gain_hist).all()
    assert (st["best_block_hist"] == ref.best_block_hist).all()
    assert st["pct_perf"] == ref.percentiles["perf"] and st["pct_gain"] == ref.percentiles["gain"]
    assert st["n_rows"] == n


def test_out_of_range_ids_rejected():
    """block ids >= n_blocks or matrix indices >= n_matrices are never used as
    histogram indices; lscat_stats reports the table as invalid (the oracle rejects it too)."""
    c = ctx()
    from paper_2103_14409_b200 import LscatError, ERR_INVALID_ARG
    for bid_bad, mat_bad in ((40, 0), (3, 9)):
        t = dict(runtime_ms=np.array([1.0, 0.5, 2.0, 1.0], np.float32),
                 block_id=np.array([0, bid_bad, 0, 31], np.uint16),
                 group_offset=np.array([0, 2, 4], np.int64),
                 group_matrix=np.array([mat_bad, 1], np.uint32))
        g_opts, _ = _opts_pair()
        c.reduce_table(_device_table(t), g_opts)
        with pytest.raises(LscatError) as e:
            c.stats(g_opts, percentiles=[0.5])
        assert e.value.status == ERR_INVALID_ARG
    # the context stays usable
    t = dict(runtime_ms=np.array([1.0, 0.5], np.float32), block_id=np.array([0, 31], np.uint16),
             group_offset=np.array([0, 2], np.int64), group_matrix=np.array([0], np.uint32))
    _compare(t)


def test_stats_after_dropping_reduce_outputs():
    """the per-group perf/gain tensors lscat_stats reads for the percentiles stay
    alive when the caller drops reduce_table's result (the binding holds them)."""
    import torch
    c = ctx()
    t = gen_table(200_000, 800, preset="t4", seed=5)
    g_opts, o_opts = _opts_pair()
    c.reduce_table(_device_table(t), g_opts)          # result dropped immediately
    junk = [torch.full((1 << 20,), 7.0, dtype=torch.float64, device="cuda") for _ in range(16)]
    torch.cuda.synchronize()
    st = c.stats(g_opts, percentiles=PCTS)
    ref = OT.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                          group_matrix=t["group_matrix"], opts=o_opts, percentiles=PCTS)
    assert st["pct_perf"] == ref.percentiles["perf"] and st["pct_gain"] == ref.percentiles["gain"]
    del junk


@pytest.mark.parametrize("seed", range(3))
def test_kernel_rollup_kernel_lengths(seed):
    """The roll-up's warp-segmented pass on kernels of 1 to ~3000 groups (within a 32-group
    chunk, across chunks, across warps' ranges, across the whole table), ragged groups with
    NaN / missing largest rows, explicit non-monotone kernel ids."""
    from tests.test_oracle_table import _random_table
    rng = np.random.default_rng(700 + seed)
    G = 40_000
    rt, bid, off, gm = _random_table(rng, G, 32, nan_p=0.1, dup_vals=False)
    lens = []
    while sum(lens) < G:
        lens.append(int(rng.choice([1, 2, 3, 7, 8, 31, 32, 33, 64, 100, 1000, 3000])))
    ids = rng.permutation(len(lens)).astype(np.uint32) * 13 + 5
    gk = np.repeat(ids, lens)[:G]
    t = dict(runtime_ms=rt, block_id=bid, group_offset=off, group_matrix=gm, group_kernel=gk)
    _compare(t, rollup=1)


def test_percentiles_sampled_first_level():
    """More than 2^20 ratio-defined groups with <= 9 percentiles take the sampled first level
    (one pass copying the keys of sample-derived intervals, exact counts below each interval):
    values exact against the oracle, ragged table, NaN groups."""
    t = gen_table(40_000_000, 150_000, preset="t4", nan_rate=0.03, seed=2024)
    _compare(t, pcts=[0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99])


def test_percentiles_sampled_fallback():
    """A sampling miss (forced: LSCAT_SEL_FORCE_MISS=1) restarts the selection on the histogram
    path, which stays exact (child process: the switch is read once)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np\n"
        "from tests.test_gpu_reduce import _compare\n"
        "from synth import gen_table\n"
        "t = gen_table(36_000_000, 140_000, preset='gtx980', nan_rate=0.03, seed=7)\n"
        "_compare(t, pcts=[0.01, 0.1, 0.5, 0.9, 0.99])\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LSCAT_SEL_FORCE_MISS="1", LSCAT_SEL_DEBUG="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
    assert "sampled 1 fail 1" in r.stderr, r.stderr[-2000:]


def _run_child(code, env_add, timeout=900):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **env_add)
    return subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                          timeout=timeout)


@pytest.mark.parametrize("knob", ["LSCAT_SEL_FIN_FORCE_FAIL", "LSCAT_SEL_NOFINISH"])
def test_percentiles_sampled_chain_after_check(knob):
    """After the sampled first level, one rank finishes the selection in one cooperative launch
    (sel_finish).  With the finisher handing over at once (forced) or switched off, the
    multi-level chain continues from the state the check left and stays exact (child process:
    the switches are read once)."""
    code = (
        "from tests.test_gpu_reduce import _compare\n"
        "from synth import gen_table\n"
        "t = gen_table(36_000_000, 140_000, preset='t4', nan_rate=0.03, seed=17)\n"
        "_compare(t, pcts=[0.01, 0.1, 0.25, 0.5, 0.9, 0.99])\n"
        "print('ok')\n")
    r = _run_child(code, {knob: "1", "LSCAT_SEL_DEBUG": "1"})
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
    assert "sampled 1 fail 0" in r.stderr, r.stderr[-2000:]
    if knob == "LSCAT_SEL_FIN_FORCE_FAIL":
        assert "sel_finish: fail 1" in r.stderr, r.stderr[-2000:]
    else:
        assert "sel_finish" not in r.stderr, r.stderr[-2000:]


def test_percentiles_sampled_finish_overflow():
    """sel_finish on a sub-bin of more than 8192 keys (~40 % of 2.5 M ratio-defined groups at
    four perf values 2^23 ulps apart: one fixed bin, one sub-bin): it hands over to the chain,
    which gathers / compacts as usual; values exact against the oracle."""
    code = (
        "import numpy as np\n"
        "from tests.test_gpu_reduce import _compare\n"
        "rng = np.random.default_rng(5)\n"
        "G = 2_500_000\n"
        "b = rng.uniform(0.5, 2.0, G).astype(np.float32)\n"
        "dense = rng.random(G) < 0.4\n"
        "j = rng.integers(1, 5, G).astype(np.float32)\n"
        "t = np.where(dense, b * (np.float32(1) + j * np.float32(2.0 ** -22)),\n"
        "             b * rng.uniform(1.0, 4.0, G).astype(np.float32)).astype(np.float32)\n"
        "rt = np.empty(2 * G, np.float32)\n"
        "rt[0::2], rt[1::2] = b, t\n"
        "tab = dict(runtime_ms=rt, block_id=np.tile(np.array([0, 1], np.uint16), G),\n"
        "           group_offset=np.arange(0, 2 * G + 1, 2, dtype=np.int64),\n"
        "           group_matrix=np.zeros(G, np.uint32))\n"
        "_compare(tab, L=2, M=1, ell=1, pcts=[0.05, 0.3, 0.5, 0.7, 0.95])\n"
        "print('ok')\n")
    r = _run_child(code, {"LSCAT_SEL_DEBUG": "1"})
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
    import re
    assert "sampled 1 fail 0" in r.stderr and re.search(r"sel_finish: fail [1-9]", r.stderr), r.stderr[-2000:]


# ---- R-27: the selection enqueued by reduce_table (percentiles in the reduce options) ------
def test_early_selection_small_tables():
    """configs[2]-shaped table: the one-launch selection enqueued right after the reducer;
    values exact against the oracle, then a different percentile list (the usual path) and
    the early list again (the early result was invalidated: the usual path, still exact)."""
    t = gen_table(2_140_796, 8363, preset="gtx980", nan_rate=0.03, seed=980)
    _compare(t, early=True)
    from paper_2103_14409_b200 import reduce_opts
    c = ctx()
    tab = _device_table(t)
    g = reduce_opts(32, 8, percentiles=PCTS)
    c.reduce_table(tab, g, per_group=False)
    other = [0.3, 0.6]
    st2 = c.stats(g, percentiles=other)
    st1 = c.stats(g, percentiles=PCTS)
    ref = OT.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                          group_matrix=t["group_matrix"], opts=OT.Opts(), percentiles=PCTS)
    ref2 = OT.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                           group_matrix=t["group_matrix"], opts=OT.Opts(), percentiles=other)
    assert st1["pct_perf"] == ref.percentiles["perf"] and st1["pct_gain"] == ref.percentiles["gain"]
    assert st2["pct_perf"] == ref2.percentiles["perf"] and st2["pct_gain"] == ref2.percentiles["gain"]


PCT9 = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]


@pytest.mark.parametrize("preset,seed", [("t4", 31), ("gtx980", 32)])
def test_early_sampled_ragged(preset, seed):
    """More than 2^20 groups with the percentiles in the reduce options: the sampled first
    level (fixed-bin intervals from a sample, one pass counting every key into its slot or gap
    and copying the slot keys, the exact check) and sel_finish enqueued behind the reducer:
    values exact against the oracle (child process: the debug switch is read once)."""
    code = (
        "from tests.test_gpu_reduce import _compare, PCT9\n"
        "from synth import gen_table\n"
        f"t = gen_table(40_000_000, 150_000, preset='{preset}', nan_rate=0.03, seed={seed})\n"
        "_compare(t, pcts=PCT9, early=True)\n"
        "print('ok')\n")
    r = _run_child(code, {"LSCAT_SEL_DEBUG": "1"})
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
    assert "sel early sampled" in r.stderr and "sampled 1 fail 0" in r.stderr, r.stderr[-2000:]
    assert "sel_finish: fail 0" in r.stderr, r.stderr[-2000:]


def test_early_sampled_uniform_table():
    """The uniform 32-row reducer (configs[4]'s kernel) with the selection enqueued behind it:
    1.5 M groups without an offset array, every counter and the values exact against the
    oracle."""
    from paper_2103_14409_b200 import reduce_opts
    c = ctx()
    n, K = 48_000_000, 187_500
    h = gen_table(n, K, preset="t4", seed=99)
    tab = _uniform_device_table(h["runtime_ms"], h["block_id"])
    g = reduce_opts(32, 8, percentiles=PCT9)
    c.reduce_table(tab, g, per_group=False)
    st = c.stats(g, percentiles=PCT9)
    ref = OT.reduce_table(h["runtime_ms"], h["block_id"], rows_per_group=32, opts=OT.Opts(),
                          percentiles=PCT9)
    for k, v in ref.counters.items():
        assert st[k] == v, (k, st[k], v)
    assert (st["perf_hist"] == ref.perf_hist).all() and (st["gain_hist"] == ref.gain_hist).all()
    assert st["pct_perf"] == ref.percentiles["perf"] and st["pct_gain"] == ref.percentiles["gain"]


def test_early_sampled_forced_miss():
    """An enqueued sampled first level that misses (forced: LSCAT_SEL_FORCE_MISS=1) makes
    lscat_stats run the histogram path over the kept perf/gain values: still exact."""
    code = (
        "from tests.test_gpu_reduce import _compare, PCT9\n"
        "from synth import gen_table\n"
        "t = gen_table(36_000_000, 140_000, preset='gtx980', nan_rate=0.03, seed=7)\n"
        "_compare(t, pcts=PCT9, early=True)\n"
        "print('ok')\n")
    r = _run_child(code, {"LSCAT_SEL_FORCE_MISS": "1", "LSCAT_SEL_DEBUG": "1"})
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
    assert "sel early sampled" in r.stderr and "sampled 1 fail 1" in r.stderr, r.stderr[-2000:]


def test_early_sampled_finish_fallback():
    """The enqueued sel_finish handing over at once (forced): the chain continues over the
    sampled pass's copies, exact."""
    code = (
        "from tests.test_gpu_reduce import _compare, PCT9\n"
        "from synth import gen_table\n"
        "t = gen_table(36_000_000, 140_000, preset='t4', nan_rate=0.03, seed=17)\n"
        "_compare(t, pcts=PCT9, early=True)\n"
        "print('ok')\n")
    r = _run_child(code, {"LSCAT_SEL_FIN_FORCE_FAIL": "1", "LSCAT_SEL_DEBUG": "1"})
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
    assert "sel early sampled" in r.stderr and "sel_finish: fail 1" in r.stderr, r.stderr[-2000:]


def test_small_table_graph_replay():
    """lscat_reduce_table on a small device table is captured on its second call with the same
    arguments and replayed as one graph afterwards: repeated calls (with and without the early
    percentiles, per-group outputs, a larger table reduced in between that reallocates the
    scratch the graph was captured against) stay exact against the oracle."""
    from paper_2103_14409_b200 import reduce_opts
    c = ctx()
    t = gen_table(300_000, 1200, preset="t4", nan_rate=0.03, seed=55)
    big = gen_table(3_000_000, 12_000, preset="gtx980", nan_rate=0.03, seed=56)
    ref = OT.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"], group_matrix=t["group_matrix"],
                          opts=OT.Opts(), percentiles=PCTS)
    tab, tab_big = _device_table(t), _device_table(big)
    for early in (True, False):
        g = reduce_opts(32, 8, **(dict(percentiles=PCTS) if early else {}))
        for i in range(5):
            if i == 3:  # grows the reducer / selection scratch: the cached graph must not be replayed
                gb = reduce_opts(32, 8, percentiles=PCTS)
                c.reduce_table(tab_big, gb, per_group=False)
                c.stats(gb, percentiles=PCTS)
            out = c.reduce_table(tab, g, per_group=(i == 4))
            st = c.stats(g, percentiles=PCTS)
            for k, v in ref.counters.items():
                assert st[k] == v, (early, i, k, st[k], v)
            assert (st["perf_hist"] == ref.perf_hist).all() and (st["gain_hist"] == ref.gain_hist).all()
            assert st["pct_perf"] == ref.percentiles["perf"] and st["pct_gain"] == ref.percentiles["gain"]
            if i == 4:
                assert (out["best_block_id"].cpu().numpy().view(np.uint16) == ref.best_block).all()
