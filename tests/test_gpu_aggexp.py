"""GPU aggregation experiment (lscat_aggregation_experiment) vs the oracle: per-repetition
aggregates bit-exact (same sampling, same sorted summation order), spreads within 1e-12."""
import numpy as np
import pytest

from oracle import aggexp as A
from synth.pool import runtime_pool
from tests.gpu_util import ctx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,reps,seed", [(10, 3000, 0), (7, 1000, 5), (1, 50, 2), (64, 200, 9)])
def test_aggregation_experiment_parity(k, reps, seed):
    import torch
    c = ctx()
    pool = runtime_pool(100_000, seed=seed)
    res = c.aggregation_experiment(torch.from_numpy(pool).cuda(), k=k, reps=reps, seed=seed,
                                   aggregates=True)
    agg, spread, means = A.experiment(pool, k=k, reps=reps, seed=seed)
    assert (res["aggregates"] == np.array(agg)).all()
    for m, name in enumerate(A.METHODS):
        assert abs(res["spread"][name] - spread[m]) <= 1e-12 * max(1.0, abs(spread[m]))
        assert abs(res["mean"][name] - means[m]) <= 1e-12 * abs(means[m])


def test_aggregation_experiment_rejects_bad_args():
    import torch
    from paper_2103_14409_b200 import LscatError
    c = ctx()
    pool = torch.ones(5, device="cuda")
    with pytest.raises(LscatError):
        c.aggregation_experiment(pool, k=10, reps=10)
    with pytest.raises(LscatError):
        c.aggregation_experiment(torch.ones(100, device="cuda"), k=65, reps=10)
