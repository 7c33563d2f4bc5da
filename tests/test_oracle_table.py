"""Pins of the C table-analysis oracle against things other than itself:

* hand-computed golden table (tests/golden/hand_table.json) and SPEC examples
  (tests/golden/spec_examples.json);
* an independent brute force written here: pandas groupby/idxmin (the paper's own tool,
  P:226) for the argmin, fractions.Fraction for every bin/threshold/fixed-point value,
  numpy sort for percentiles;
* invariants: histogram sums, scale invariance by 2^k, row permutation within
  groups, the identity gain > 1/5 <=> perf < 5/6, planted-best recovery.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pandas as pd
import pytest

from synth import gen_table

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _table_from_groups(groups):
    rt, bid, off = [], [], [0]
    for g in groups:
        for b, v in enumerate(g["runtime"]):
            rt.append(float("nan") if v == "nan" else float(v))
            bid.append(b)
        off.append(len(rt))
    return (np.array(rt, np.float32), np.array(bid, np.uint16), np.array(off, np.int64),
            np.array([g["matrix"] for g in groups], np.uint32))


def test_hand_golden(oracle_lib):
    G = json.load(open(os.path.join(GOLDEN, "hand_table.json")))
    rt, bid, off, gm = _table_from_groups(G["groups"])
    o = oracle_lib.Opts(n_blocks=G["n_blocks"], largest_block_id=G["largest_block_id"],
                        n_matrices=G["n_matrices"])
    E = G["expected_skipna"]
    r = oracle_lib.reduce_table(rt, bid, off, group_matrix=gm, opts=o,
                                percentiles=E["percentiles"]["p"])
    for k, v in E["counters"].items():
        assert r.counters[k] == v, k
    assert list(r.best_block) == E["best_block"]
    nz = {str(i): int(c) for i, c in enumerate(r.perf_hist) if c}
    assert nz == E["perf_hist_nonzero"]
    nz = {str(i): int(c) for i, c in enumerate(r.gain_hist) if c}
    assert nz == E["gain_hist_nonzero"]
    assert r.best_block_hist.tolist() == E["best_block_hist"]
    assert abs(r.derived["mean_perf"] - E["mean_perf_approx"]) < 1e-15
    assert r.derived["mean_gain"] == E["mean_gain"]
    assert r.percentiles["perf"] == E["percentiles"]["perf"]
    assert r.percentiles["gain"] == E["percentiles"]["gain"]
    r2 = oracle_lib.reduce_table(rt, bid, off, group_matrix=gm,
                                 opts=oracle_lib.Opts(n_blocks=4, largest_block_id=3,
                                                      n_matrices=2, nan_policy=1))
    for k, v in G["expected_complete_only"]["counters"].items():
        assert r2.counters[k] == v, k


def test_spec_examples(oracle_lib):
    S = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))
    for c in S["cases"]:
        thr = c["threads"]
        rt = np.array(c["runtime"], np.float32)
        o = oracle_lib.Opts(n_blocks=len(thr), largest_block_id=len(thr) - 1, n_matrices=1)
        r = oracle_lib.reduce_table(rt, np.arange(len(thr)), np.array([0, len(thr)]), opts=o)
        if "best_threads" in c:
            assert thr[r.best_block[0]] == c["best_threads"], c["spec"]
        if "perf_bin" in c:
            assert r.perf_hist[c["perf_bin"]] == 1, c["spec"]
            assert r.perf[0] == c["perf"], c["spec"]
        if "gain_bin" in c:
            assert r.gain_hist[c["gain_bin"]] == 1, c["spec"]
            assert bool(r.flags[0] & 0x40) == c["gain_gt"], c["spec"]


# ----------------------------------------------------------------------------------------
# Independent brute force (pandas + Fraction)
# ----------------------------------------------------------------------------------------
def brute_force(rt, bid, off, gm, L, ell, nb=100, cap=10, policy=0, n_matrices=8):
    df = pd.DataFrame({"g": np.repeat(np.arange(len(off) - 1), np.diff(off)),
                       "b": bid.astype(np.int64), "r": rt.astype(np.float64)})
    ok = np.isfinite(df.r) & (df.r > 0)
    res = dict(n_rows=len(df), n_ok=int(ok.sum()), n_nan=int(np.isnan(df.r).sum()))
    res["n_invalid"] = res["n_rows"] - res["n_ok"] - res["n_nan"]
    dok = df[ok].sort_values(["g", "b"])
    # pandas: min skips NaN; idxmin -> first occurrence in block order = smaller block on ties
    mins = dok.groupby("g").r.min()
    arg = dok.loc[dok.groupby("g").r.idxmin()].set_index("g").b
    cnt = df.groupby("g").size().reindex(range(len(off) - 1), fill_value=0)
    cok = dok.groupby("g").size().reindex(range(len(off) - 1), fill_value=0)
    lrow = df[df.b == ell].set_index("g").r
    perf_h = [0] * (nb + 1)
    gain_h = [0] * (cap * nb + 1)
    bbh = np.zeros((n_matrices, L), np.int64)
    c = dict(n_defined=0, n_all_nan=0, n_complete=0, n_incomplete=0, n_largest_missing=0,
             n_ratio_defined=0, n_largest_is_best=0, n_largest_strictly_slower=0, n_gain_gt=0,
             n_perf_lt=0, n_perf_band=0)
    fxp = fxg = 0
    perfs, gains, best = [], [], []
    for g in range(len(off) - 1):
        complete = cnt[g] == L and cok[g] == cnt[g]
        defined = complete if policy else cok[g] >= 1
        c["n_all_nan"] += cok[g] == 0
        c["n_complete"] += complete
        c["n_incomplete"] += not complete
        if not defined:
            best.append(0xFFFF)
            continue
        c["n_defined"] += 1
        bb = int(arg[g])
        best.append(bb)
        bbh[gm[g], bb] += 1
        if g not in lrow.index or not (np.isfinite(lrow[g]) and lrow[g] > 0):
            c["n_largest_missing"] += 1
            continue
        c["n_ratio_defined"] += 1
        B, T = Fraction(float(mins[g])), Fraction(float(lrow[g]))
        perf, gain = B / T, T / B - 1
        c["n_largest_is_best"] += bb == ell
        c["n_largest_strictly_slower"] += T > B
        c["n_gain_gt"] += gain > Fraction(1, 5)
        c["n_perf_lt"] += perf < Fraction(17, 20)
        c["n_perf_band"] += Fraction(2, 5) <= perf < Fraction(17, 20)
        perf_h[math.floor(perf * nb)] += 1
        gain_h[cap * nb if gain >= cap else math.floor(gain * nb)] += 1
        pf = float(mins[g]) / float(lrow[g])          # the stored double: RN(b / t)
        gf = float(lrow[g]) / float(mins[g]) - 1.0    # RN(RN(t / b) - 1)
        fxp += math.floor(Fraction(pf) * 2 ** 52)
        fxg += math.floor(min(Fraction(gf), Fraction(2 ** 20)) * 2 ** 32)
        perfs.append(pf)
        gains.append(gf)
    res.update(c)
    return res, perf_h, gain_h, bbh, fxp, fxg, np.array(best), np.array(perfs), np.array(gains)


def _random_table(rng, G, L, nan_p=0.1, ragged=True, dup_vals=True):
    rts, bids, off = [], [], [0]
    for g in range(G):
        n = int(rng.integers(0, L + 1)) if ragged and rng.random() < 0.2 else L
        blocks = rng.permutation(L)[:n]
        if dup_vals:
            vals = rng.choice(np.array([1.0, 1.25, 1.5, 2.0, 3.0, 0.75], np.float32), size=n)
            vals = vals * np.float32(2.0 ** rng.integers(-3, 4))
        else:
            vals = rng.uniform(0.1, 3.0, size=n).astype(np.float32)
        vals = np.where(rng.random(n) < nan_p, np.float32(np.nan), vals)
        if rng.random() < 0.05 and n:
            vals[0] = rng.choice([np.inf, -1.0, 0.0])
        rts += list(vals)
        bids += list(blocks)
        off.append(len(rts))
    return (np.array(rts, np.float32), np.array(bids, np.uint16), np.array(off, np.int64),
            rng.integers(0, 8, size=G).astype(np.uint32))


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("policy", [0, 1])
def test_brute_force(oracle_lib, seed, policy):
    rng = np.random.default_rng(seed)
    L = [4, 8, 32][seed % 3]
    ell = L - 1 if seed % 2 == 0 else L // 2
    rt, bid, off, gm = _random_table(rng, 300, L, dup_vals=seed < 3)
    o = oracle_lib.Opts(n_blocks=L, largest_block_id=ell, nan_policy=policy)
    r = oracle_lib.reduce_table(rt, bid, off, group_matrix=gm, opts=o,
                                percentiles=[0.01, 0.1, 0.5, 0.9, 0.99])
    res, ph, gh, bbh, fxp, fxg, best, perfs, gains = brute_force(rt, bid, off, gm, L, ell,
                                                                 policy=policy)
    for k, v in res.items():
        assert r.counters[k] == v, k
    assert r.perf_hist.tolist() == ph
    assert r.gain_hist.tolist() == gh
    assert (r.best_block_hist == bbh).all()
    assert (r.best_block == best).all()
    assert (r.counters["perf_fx_hi"] << 21) + r.counters["perf_fx_lo"] == fxp
    assert (r.counters["gain_fx_hi"] << 21) + r.counters["gain_fx_lo"] == fxg
    for i, p in enumerate([0.01, 0.1, 0.5, 0.9, 0.99]):
        n = len(perfs)
        k = min(max(int(np.ceil(p * n)), 1), n)
        assert r.percentiles["perf"][i] == np.sort(perfs)[k - 1]
        assert r.percentiles["gain"][i] == np.sort(gains)[k - 1]
    # exact means from the fixed-point totals equal the Fraction mean within the truncation
    if res["n_ratio_defined"]:
        exact = sum(Fraction(p) for p in perfs) / len(perfs)
        assert abs(Fraction(r.derived["mean_perf"]) - exact) <= Fraction(1, 2 ** 50)
    _check_finalize(r.derived, res, fxp, fxg)


def _ulp(x):
    return math.ulp(x) if x else 2.0 ** -1074


def _check_finalize(D, res, fxp, fxg):
    """a10 / oracle_finalize pinned by exact rationals: every fraction is the
    correctly rounded count / denominator with the denominators of O3 step 11 -- n_rows for
    frac_nonnan, n_ratio_defined for every other share (groups
    whose largest-block row is missing or NaN are excluded, R-7/R-9) -- and each mean is the
    brute-force fixed-point total / (2^s n_ratio_defined) within one ulp (O3 step 9)."""
    nrd = res["n_ratio_defined"]
    assert D["frac_nonnan"] == float(Fraction(res["n_ok"], res["n_rows"]))
    if nrd == 0:
        for k in ("frac_largest_not_best", "frac_gain_gt", "frac_perf_lt", "frac_perf_band",
                  "mean_perf", "mean_gain"):
            assert math.isnan(D[k]), k
        return
    assert D["frac_largest_not_best"] == float(Fraction(nrd - res["n_largest_is_best"], nrd))
    assert D["frac_gain_gt"] == float(Fraction(res["n_gain_gt"], nrd))
    assert D["frac_perf_lt"] == float(Fraction(res["n_perf_lt"], nrd))
    assert D["frac_perf_band"] == float(Fraction(res["n_perf_band"], nrd))
    mp = Fraction(fxp, 2 ** 52 * nrd)
    mg = Fraction(fxg, 2 ** 32 * nrd)
    assert abs(Fraction(D["mean_perf"]) - mp) <= Fraction(_ulp(float(mp)))
    assert abs(Fraction(D["mean_gain"]) - mg) <= Fraction(_ulp(float(mg)))


def test_finalize_denominators_distinguishable(oracle_lib):
    """The random tables of test_brute_force make every denominator choice observable: groups
    that are defined but lack a usable largest-block row (n_defined > n_ratio_defined), and
    largest-is-best groups, so a wrong denominator or numerator changes a fraction."""
    rng = np.random.default_rng(0)
    rt, bid, off, gm = _random_table(rng, 300, 4, dup_vals=True)
    r = oracle_lib.reduce_table(rt, bid, off, group_matrix=gm,
                                opts=oracle_lib.Opts(n_blocks=4, largest_block_id=3))
    C, D = r.counters, r.derived
    assert C["n_defined"] > C["n_ratio_defined"] > C["n_largest_is_best"] > 0
    assert C["n_ratio_defined"] > C["n_perf_lt"] > 0 and C["n_perf_band"] > 0
    wrong = float(Fraction(C["n_defined"] - C["n_largest_is_best"], C["n_defined"]))
    assert D["frac_largest_not_best"] != wrong
    assert D["frac_perf_lt"] != float(Fraction(C["n_perf_lt"], C["n_defined"]))


def test_invariants_generator_table(oracle_lib):
    t = gen_table(200_000, 800, preset="t4", nan_rate=0.03, seed=7, return_planted=True)
    o = oracle_lib.Opts()
    r = oracle_lib.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                                group_matrix=t["group_matrix"], opts=o)
    C = r.counters
    assert C["n_ok"] + C["n_nan"] + C["n_invalid"] == C["n_rows"]
    assert int(r.perf_hist.sum()) == C["n_ratio_defined"]
    assert int(r.gain_hist.sum()) == C["n_ratio_defined"]
    assert int(r.best_block_hist.sum()) == C["n_defined"]
    assert C["n_defined"] == C["n_ratio_defined"] + C["n_largest_missing"]
    rd = (r.flags & 0x8) != 0
    assert (r.perf[rd] <= 1.0).all() and (r.perf[rd] > 0).all()
    # identity: gain > 1/5  <=>  perf < 5/6  (exact predicates)
    o56 = oracle_lib.Opts(perf_lt=(5, 6))
    r56 = oracle_lib.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                                  group_matrix=t["group_matrix"], opts=o56)
    assert ((r.flags & 0x40) != 0).tolist() == ((r56.flags & 0x80) != 0).tolist()
    # planted best recovered wherever the planted row has a result
    G = t["n_groups"]
    off = t["group_offset"]
    for g in range(0, G, 7):
        rows = slice(off[g], off[g + 1])
        b = t["block_id"][rows]
        v = t["runtime_ms"][rows]
        pl = t["planted"][g]
        if (b == pl).any() and np.isfinite(v[b == pl][0]):
            assert r.best_block[g] == pl


def test_scale_and_permutation_invariance(oracle_lib):
    t = gen_table(50_000, 200, preset="gtx980", nan_rate=0.05, seed=3)
    base = oracle_lib.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                                   group_matrix=t["group_matrix"], percentiles=[0.1, 0.5])
    for k in (-5, 3):
        s = oracle_lib.reduce_table(t["runtime_ms"] * np.float32(2.0 ** k), t["block_id"],
                                    t["group_offset"], group_matrix=t["group_matrix"],
                                    percentiles=[0.1, 0.5])
        assert s.counters == base.counters
        assert (s.perf_hist == base.perf_hist).all() and (s.gain_hist == base.gain_hist).all()
        assert (s.best_block == base.best_block).all()
        assert s.percentiles == base.percentiles
    rng = np.random.default_rng(1)
    rt, bid = t["runtime_ms"].copy(), t["block_id"].copy()
    off = t["group_offset"]
    for g in range(t["n_groups"]):
        p = off[g] + rng.permutation(off[g + 1] - off[g])
        rt[off[g]:off[g + 1]], bid[off[g]:off[g + 1]] = rt[p], bid[p]
    s = oracle_lib.reduce_table(rt, bid, off, group_matrix=t["group_matrix"],
                                percentiles=[0.1, 0.5])
    assert s.counters == base.counters and s.percentiles == base.percentiles
    assert (s.best_block == base.best_block).all()


def test_shard_merge_invariance(oracle_lib):
    """Group-aligned shards reduced separately and summed give the same integers (a9)."""
    t = gen_table(60_000, 300, preset="t4", seed=11)
    full = oracle_lib.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                                   group_matrix=t["group_matrix"])
    G = t["n_groups"]
    for W in (2, 3, 8):
        tot = {k: 0 for k in full.counters}
        ph = np.zeros_like(full.perf_hist)
        for r in range(W):
            g0, g1 = G * r // W, G * (r + 1) // W
            s = gen_table(60_000, 300, preset="t4", seed=11, group_begin=g0, group_end=g1)
            part = oracle_lib.reduce_table(s["runtime_ms"], s["block_id"],
                                           s["group_offset"], group_matrix=s["group_matrix"])
            for k in tot:
                tot[k] += part.counters[k]
            ph += part.perf_hist
        assert tot == full.counters
        assert (ph == full.perf_hist).all()


def test_duplicate_rows_rejected(oracle_lib):
    with pytest.raises(oracle_lib.OracleError):
        oracle_lib.reduce_table(np.array([1, 2], np.float32), np.array([0, 0]),
                                np.array([0, 2]), opts=oracle_lib.Opts(n_blocks=2))


def test_block_profile_brute_force(oracle_lib):
    """R-22 block profile == Fraction brute force: per (matrix, block) floor(RN(best/r)*2^31)."""
    rng = np.random.default_rng(5)
    rt, bid, off, gm = _random_table(rng, 400, 8, dup_vals=False)
    r = oracle_lib.reduce_table(rt, bid, off, group_matrix=gm,
                                opts=oracle_lib.Opts(n_blocks=8, block_profile=True))
    ps = np.zeros((8, 8), object)
    pc = np.zeros((8, 8), np.int64)
    for g in range(len(off) - 1):
        rows = range(off[g], off[g + 1])
        okr = [i for i in rows if np.isfinite(rt[i]) and rt[i] > 0]
        if not okr:
            continue
        best = min(float(rt[i]) for i in okr)
        for i in okr:
            q = float(best) / float(rt[i])                    # RN(best / r)
            ps[gm[g], bid[i]] += math.floor(Fraction(q) * 2 ** 31)
            pc[gm[g], bid[i]] += 1
    assert (r.profile_count == pc).all()
    assert all(int(r.profile_sum[i, j]) == int(ps[i, j]) for i in range(8) for j in range(8))
    # the best block of a group with a unique minimum contributes exactly 2^31 (perf 1)
    assert r.profile_mean.max() <= 1.0


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_parallel_oracle_equals_oracle(oracle_lib, threads):
    """The all-cores baseline variant (group-aligned chunks, integer partials summed) gives the
    single-threaded oracle's counters and histograms exactly, ragged and uniform tables."""
    rng = np.random.default_rng(threads)
    rt, bid, off, gm = _random_table(rng, 500, 8, dup_vals=True)
    o = oracle_lib.Opts(n_blocks=8)
    r = oracle_lib.reduce_table(rt, bid, off, group_matrix=gm, opts=o)
    c, ph, gh, bh = oracle_lib.reduce_table_parallel(rt, bid, off, group_matrix=gm, opts=o,
                                                     threads=threads)
    assert c == r.counters and (ph == r.perf_hist).all() and (gh == r.gain_hist).all()
    assert (bh == r.best_block_hist).all()
    t = gen_table(32 * 1000 - 7, 125, preset="t4", seed=3)
    r = oracle_lib.reduce_table(t["runtime_ms"], t["block_id"], rows_per_group=32, first_group=5)
    c, ph, gh, bh = oracle_lib.reduce_table_parallel(t["runtime_ms"], t["block_id"],
                                                     rows_per_group=32, first_group=5,
                                                     threads=threads)
    assert c == r.counters and (ph == r.perf_hist).all() and (bh == r.best_block_hist).all()


# ----------------------------------------------------------------------------------------
# Per-kernel roll-up (R-26)
# ----------------------------------------------------------------------------------------
def test_kernel_rollup_golden(oracle_lib):
    g = json.load(open(os.path.join(GOLDEN, "kernel_rollup.json")))
    rt, bid, off, gm = _table_from_groups(g["groups"])
    gk = np.array([x["kernel"] for x in g["groups"]], np.uint32)
    o = oracle_lib.Opts(n_blocks=g["n_blocks"], n_matrices=g["n_matrices"])
    r = oracle_lib.reduce_table(rt, bid, off, group_matrix=gm, opts=o, group_kernel=gk,
                                kernel_rollup=True)
    e = g["expected"]
    for k in ("n_kernels", "n_kernels_not_best", "n_kernels_perf_lt", "n_kernels_perf_band"):
        assert r.rollup[k] == e[k], k
    # sum over kernels of floor(S_k / c_k) = the four per-kernel values listed in the golden
    assert sum(e["kernel_mean_fx"].values()) == e["kernel_mean_fx_total"]
    assert (r.rollup["kernel_mean_fx_hi"] << 21) + r.rollup["kernel_mean_fx_lo"] == e["kernel_mean_fx_total"]
    want = np.zeros(101, np.uint64)
    for b, v in e["perf_hist_nonzero"].items():
        want[int(b)] = v
    assert (r.rollup["perf_hist"] == want).all()
    assert r.rollup["frac_kernels_not_best"] == 3 / 4
    assert r.rollup["frac_kernels_perf_band"] == 2 / 4
    # the roll-up does not depend on the order of the groups (the oracle sorts by kernel id)
    perm = np.random.default_rng(0).permutation(len(g["groups"]))
    rt2, bid2, off2, gm2 = _table_from_groups([g["groups"][i] for i in perm])
    r2 = oracle_lib.reduce_table(rt2, bid2, off2, group_matrix=gm2, opts=o, group_kernel=gk[perm],
                                 kernel_rollup=True)
    assert {k: r2.rollup[k] for k in e if k in r2.rollup} == {k: r.rollup[k] for k in e if k in r.rollup}


@pytest.mark.parametrize("seed", range(4))
def test_kernel_rollup_brute_force(oracle_lib, seed):
    """Fraction brute force of every roll-up quantity from the brute-force per-group values
    (pandas argmin, Fraction-free RN(b/t) doubles) on random ragged tables with contiguous
    kernels of 1..10 groups."""
    rng = np.random.default_rng(100 + seed)
    L = [4, 8, 32][seed % 3]
    ell = L - 1
    G = 400
    rt, bid, off, gm = _random_table(rng, G, L, dup_vals=seed < 2)
    sizes = rng.integers(1, 11, G)
    gk = np.repeat(np.arange(G), sizes)[:G].astype(np.uint32) * 7 + 3
    o = oracle_lib.Opts(n_blocks=L, largest_block_id=ell)
    r = oracle_lib.reduce_table(rt, bid, off, group_matrix=gm, opts=o, group_kernel=gk,
                                kernel_rollup=True)
    res, ph, gh, bbh, fxp, fxg, best, perfs, gains = brute_force(rt, bid, off, gm, L, ell)
    # per-group ratio-defined flag and perf, recomputed independently
    df_ok = np.isfinite(rt) & (rt > 0)
    per = {}
    for g in range(G):
        rows = range(off[g], off[g + 1])
        okr = [i for i in rows if df_ok[i]]
        lrow = [i for i in rows if bid[i] == ell]
        if not okr or not lrow or not df_ok[lrow[0]]:
            continue
        b = min(float(rt[i]) for i in okr)
        t = float(rt[lrow[0]])
        per.setdefault(int(gk[g]), []).append((math.floor(Fraction(b / t) * 2 ** 52), best[g] != ell))
    n_k = len(per)
    nb_ = sum(any(x[1] for x in v) for v in per.values())
    lt = band = 0
    hist = [0] * 101
    mean_fx = 0
    for v in per.values():
        S, c = sum(x[0] for x in v), len(v)
        P = Fraction(S, c * 2 ** 52)
        lt += P < Fraction(17, 20)
        band += Fraction(2, 5) <= P < Fraction(17, 20)
        hist[math.floor(P * 100)] += 1
        mean_fx += S // c
    R = r.rollup
    assert R["n_kernels"] == n_k and R["n_kernels_not_best"] == nb_
    assert R["n_kernels_perf_lt"] == lt and R["n_kernels_perf_band"] == band
    assert R["perf_hist"].tolist() == hist
    assert (R["kernel_mean_fx_hi"] << 21) + R["kernel_mean_fx_lo"] == mean_fx
    assert n_k >= nb_ > 0
