"""lscat_ingest groups an unordered dataframe into a table.  Oracle: a stable
numpy lexsort (the definition: groups by (kernel, matrix) ascending, rows by block id, ties
in input order); the reduced statistics must then equal those of the generator's table."""
import numpy as np
import pytest

from oracle import table as OT
from synth import gen_table
from tests.gpu_util import ctx

pytestmark = pytest.mark.gpu


def _shuffled(t, seed):
    rng = np.random.default_rng(seed)
    G = t["n_groups"]
    gk = np.repeat(t["group_kernel"], np.diff(t["group_offset"]))
    gm = np.repeat(t["group_matrix"], np.diff(t["group_offset"]))
    p = rng.permutation(t["n_rows"])
    return gk[p], gm[p], t["block_id"][p], t["runtime_ms"][p], t["status"][p]


@pytest.mark.parametrize("n,K,seed", [(1000, 10, 1), (2_140_796, 8363, 980), (100_000, 90_000, 3)])
def test_ingest_matches_lexsort(n, K, seed):
    import torch
    c = ctx()
    t = gen_table(n, K, preset="gtx980", seed=seed)
    gk, gm, bid, rt, st = _shuffled(t, seed)
    T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()
    tab = c.ingest(T(gk.astype(np.uint32), np.int32), T(gm.astype(np.uint32), np.int32),
                   T(bid, np.int16), T(rt, np.float32), T(st, np.uint8))
    out = tab.to_numpy()
    order = np.lexsort((bid, gm, gk))                      # stable: last key primary
    assert out["n_rows"] == n
    assert (out["runtime_ms"].view(np.uint32) == rt[order].view(np.uint32)).all()
    assert (out["block_id"] == bid[order]).all()
    assert (out["status"] == st[order]).all()
    keys = gk[order].astype(np.int64) * 1_000_000 + gm[order]
    starts = np.r_[0, np.nonzero(np.diff(keys))[0] + 1]
    assert out["n_groups"] == len(starts)
    assert (out["group_offset"][:-1] == starts).all() and out["group_offset"][-1] == n
    assert (out["group_kernel"] == gk[order][starts]).all()
    assert (out["group_matrix"] == gm[order][starts]).all()
    # the ingested table reduces to the same statistics as the generator's (P:226 dataframe)
    a = OT.reduce_table(out["runtime_ms"], out["block_id"], out["group_offset"],
                        group_matrix=out["group_matrix"])
    b = OT.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                        group_matrix=t["group_matrix"])
    assert a.counters == b.counters


def test_ingest_duplicates_and_empty():
    import torch
    from paper_2103_14409_b200 import LscatError
    c = ctx()
    k = torch.tensor([3, 1, 3, 1], dtype=torch.int32, device="cuda")
    m = torch.tensor([0, 2, 0, 2], dtype=torch.int32, device="cuda")
    b = torch.tensor([5, 1, 5, 0], dtype=torch.int16, device="cuda")
    r = torch.tensor([1.0, 2.0, 3.0, 4.0], device="cuda")
    with pytest.raises(LscatError):
        c.ingest(k, m, b, r)
    e = torch.empty(0, device="cuda")
    tab = c.ingest(e.int(), e.int(), e.short(), e)
    assert tab.n_rows == 0 and tab.n_groups == 0
