"""CPU oracle of the aggregation experiment (R-23).  TEST INFRASTRUCTURE ONLY.

Plain Python integers/floats, step by step: Floyd's sampling without replacement driven by the
counter-based generator both sides implement (splitmix64), the five aggregates of the sorted
sample (sums in ascending order, one rounding per addition), and the variation of each method
= population standard deviation of its aggregates / their mean (sequential sums).
"""
from __future__ import annotations

import math

M64 = (1 << 64) - 1
METHODS = ("mean", "median", "min", "max", "trimmed_mean_20")


def splitmix64(z):
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def draw(seed, rep, j, m):
    """Uniform integer in [0, m]: multiply-shift of 32 random bits."""
    h = splitmix64(splitmix64(seed ^ ((rep * 0xD1B54A32D192ED03) & M64)) ^ j)
    return ((h >> 32) * (m + 1)) >> 32


def floyd_sample(seed, rep, n, k):
    """Floyd's algorithm: for j = n-k .. n-1 take t in [0, j], or j if t was taken."""
    idx = []
    for i in range(k):
        j = n - k + i
        t = draw(seed, rep, j, j)
        idx.append(j if t in idx else t)
    return idx


def aggregate(values):
    """The five methods on one sample: values already float (exact fp32)."""
    v = sorted(values)
    k = len(v)
    s = 0.0
    for x in v:
        s += x
    mean = s / k
    median = v[k // 2] if k % 2 else (v[k // 2 - 1] + v[k // 2]) * 0.5
    cut = k // 10
    st = 0.0
    for x in v[cut:k - cut]:
        st += x
    trimmed = st / (k - 2 * cut)
    return [mean, median, v[0], v[-1], trimmed]


def experiment(pool, k=10, reps=10_000, seed=0):
    """Returns (aggregates[5][reps], spread[5], mean[5])."""
    pool = [float(x) for x in pool]
    n = len(pool)
    agg = [[0.0] * reps for _ in range(5)]
    for r in range(reps):
        a = aggregate([pool[i] for i in floyd_sample(seed, r, n, k)])
        for m in range(5):
            agg[m][r] = a[m]
    spread, means = [], []
    for m in range(5):
        s = 0.0
        for x in agg[m]:
            s += x
        mean = s / reps
        q = 0.0
        for x in agg[m]:
            q += (x - mean) * (x - mean)
        means.append(mean)
        spread.append(math.sqrt(q / reps) / mean)
    return agg, spread, means
