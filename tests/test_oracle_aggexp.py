"""Pins of the aggregation-experiment oracle (oracle/aggexp.py)."""
import math
from collections import Counter

import numpy as np
import pytest

from oracle import aggexp as A
from synth.pool import runtime_pool


def test_aggregate_spec_examples():
    assert A.aggregate([1.0, 2.0, 3.0, 4.0, 5.0])[1] == 3.0            # S:318 median
    assert A.aggregate([1.0, 2.0, 3.0, 4.0])[1] == 2.5                 # S:319 even -> midpoint
    assert A.aggregate([1.0] * 9 + [100.0])[4] == 1.0                  # S:320 trimmed mean
    a = A.aggregate([4.0, 1.0, 3.0, 2.0])
    assert a[0] == 2.5 and a[2] == 1.0 and a[3] == 4.0


def test_floyd_sampling():
    for rep in range(50):
        s = A.floyd_sample(7, rep, 1000, 10)
        assert len(set(s)) == 10 and all(0 <= i < 1000 for i in s)
    assert sorted(A.floyd_sample(1, 3, 10, 10)) == list(range(10))   # k == n: a permutation
    c = Counter()
    for rep in range(4000):
        c.update(A.floyd_sample(11, rep, 20, 5))
    exp = 4000 * 5 / 20
    chi2 = sum((c[i] - exp) ** 2 / exp for i in range(20))
    assert chi2 < 45                                                   # 19 dof, p ~ 1e-3


def test_constant_pool_and_scale_equivariance():
    agg, spread, _ = A.experiment([5.0] * 1000, k=10, reps=200, seed=1)
    assert spread == [0.0] * 5
    pool = runtime_pool(5000, seed=3)
    a1, s1, m1 = A.experiment(pool, k=10, reps=300, seed=2)
    a2, s2, m2 = A.experiment(pool * np.float32(4.0), k=10, reps=300, seed=2)
    assert all(x * 4.0 == y for r1, r2 in zip(a1, a2) for x, y in zip(r1, r2))
    assert s1 == s2


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_median_is_most_stable(seed):
    """on a right-skewed pool with 2 % outliers the median's spread is below the mean's
    and the max's, and below 2 % ("variation of around one percent")."""
    pool = runtime_pool(100_000, seed=seed)
    _, spread, _ = A.experiment(pool, k=10, reps=10_000, seed=seed)
    sp = dict(zip(A.METHODS, spread))
    assert sp["median"] < sp["mean"] and sp["median"] < sp["max"]
    assert sp["median"] < 0.02


@pytest.mark.parametrize("reps", [2, 3, 50])
def test_spread_is_population_sd_over_mean(reps):
    """R-23 / S:324-332: variation = population standard deviation (ddof = 0) of the reps
    aggregates divided by their mean, recomputed here with numpy from the oracle's own
    per-repetition aggregates.  Small reps make ddof = 1 differ by sqrt(reps / (reps - 1))."""
    pool = runtime_pool(2000, seed=4)
    agg, spread, means = A.experiment(pool, k=10, reps=reps, seed=9)
    for m in range(5):
        a = np.array(agg[m], np.float64)
        assert math.isclose(means[m], a.mean(), rel_tol=1e-12)
        ref = np.std(a, ddof=0) / np.mean(a)
        assert math.isclose(spread[m], ref, rel_tol=1e-9, abs_tol=1e-15), (m, spread[m], ref)
        if np.std(a) > 0:
            assert not math.isclose(spread[m], np.std(a, ddof=1) / np.mean(a), rel_tol=1e-6)


def test_whole_pool_sample_has_no_spread():
    """k = n: every repetition samples the whole pool (a permutation), so every aggregate is
    the pool's own statistic and each variation is exactly 0."""
    pool = [3.0, 1.0, 4.0, 1.5, 9.0, 2.5, 6.0, 5.0, 3.5, 8.0]
    agg, spread, means = A.experiment(pool, k=10, reps=20, seed=1)
    s = sorted(pool)
    assert spread == [0.0] * 5
    assert means[1] == (s[4] + s[5]) / 2 and means[2] == 1.0 and means[3] == 9.0
    assert math.isclose(means[0], sum(pool) / 10) and math.isclose(means[4], sum(s[1:9]) / 8)
