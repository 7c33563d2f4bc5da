"""Runtime pool for the aggregation experiment: 100 000 positive runtimes,
right-skewed (gamma body) with 2 % large outliers (x U(2, 10)).  Input generator only."""
import numpy as np


def runtime_pool(n=100_000, seed=0, outlier_rate=0.02):
    rng = np.random.default_rng(seed)
    body = 1.0 + rng.gamma(shape=2.0, scale=0.01, size=n)
    out = rng.random(n) < outlier_rate
    body[out] *= rng.uniform(2.0, 10.0, size=int(out.sum()))
    return body.astype(np.float32)
