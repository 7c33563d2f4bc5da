"""SURVEY 8(f) #4 side analyses on the device: the occupancy-calculator block (P:230-231,
P:309) and the timeout-economics curve, against host recomputations."""
import numpy as np
import pytest

from oracle import table as OT
from synth import gen_table
from tests.gpu_util import ctx

pytestmark = pytest.mark.gpu

BLOCKS = list(range(32, 1025, 32))


def _device():
    import torch
    from oracle import occupancy as O
    p = torch.cuda.get_device_properties(0)
    d = O.Device()
    d.max_threads_per_sm = p.max_threads_per_multi_processor
    d.regs_per_sm = p.regs_per_multiprocessor
    d.smem_per_sm = p.shared_memory_per_multiprocessor
    return d


def test_occupancy_block():
    """The library's occupancy-API numbers against the oracle's restatement of the occupancy
    rule (oracle/occupancy.py) from the same compiled attributes (registers, static shared
    memory) and the device limits: blocks per SM of every candidate of every suite kernel, and
    the family choice (most resident warps, ties -> larger block)."""
    from oracle import occupancy as O
    from paper_2103_14409_b200 import KERNELS, LscatError
    c = ctx()
    dev = _device()
    for name, k in KERNELS.items():
        r = c.occupancy_block(k, BLOCKS)
        info = r["info"]
        cands = []
        for b, x in zip(BLOCKS, info):
            assert x["threads"] == b
            if x["regs_per_thread"] == 0 and x["blocks_per_sm"] == 0:   # no implementation
                cands.append((b, -1, 0, 0))
                continue
            want = O.blocks_per_sm(b, x["regs_per_thread"], x["static_smem"], x["dynamic_smem"], dev)
            assert x["blocks_per_sm"] == want, (name, b, x, want)
            assert x["warps_per_sm"] == want * b // 32
            assert 0 < x["api_block"] <= b and x["api_min_grid"] > 0, (name, b, x)
            assert x["max_threads_per_block"] >= b
            cands.append((b, x["regs_per_thread"], x["static_smem"], x["dynamic_smem"]))
        assert r["block_id"] == O.choose(cands, dev), (name, r["block_id"], O.choose(cands, dev))
        if name == "gemm_bf16":
            assert all(x["blocks_per_sm"] == 0 for x in info[:3])     # < 128 threads: none
    with pytest.raises(LscatError):
        c.occupancy_block(KERNELS["euclid"], [33])


def test_occupancy_block_quality_via_reduce():
    """The occupancy choice is evaluated like the paper's largest block: reduce the table with
    largest_block_id = that choice and compare with the oracle."""
    from paper_2103_14409_b200 import KERNELS, reduce_opts
    c = ctx()
    bid = c.occupancy_block(KERNELS["euclid"], BLOCKS)["block_id"]
    t = gen_table(100_000, 400, preset="t4", seed=3)
    from tests.test_gpu_reduce import _device_table
    o = reduce_opts(32, 8, largest_block_id=bid)
    c.reduce_table(_device_table(t), o, per_group=False)
    st = c.stats(o)
    ref = OT.reduce_table(t["runtime_ms"], t["block_id"], t["group_offset"],
                          group_matrix=t["group_matrix"], opts=OT.Opts(largest_block_id=bid))
    for k, v in ref.counters.items():
        assert st[k] == v, k


def test_timeout_curve():
    c = ctx()
    tab = c.gen_table(500_000, 2000, preset=0, seed=8)
    h = tab.to_numpy()
    taus = [1e-3, 0.01, 0.1, 0.5, 1.0, 2.0, 10.0, 30.0, 120.0]
    for (W, K, R) in [(1, 10, 1000), (1, 5, 20)]:
        got = c.timeout_curve(tab, taus, W, K, R)
        rt = h["runtime_ms"]
        ok = np.isfinite(rt) & (rt > 0)
        t = (np.float64(W + K * R) * rt.astype(np.float64)) * 1e-3
        want = [int((ok & (t <= x)).sum()) for x in taus]
        assert got.tolist() == want
        assert got[-1] <= ok.sum() and (np.diff(got.astype(np.int64)) >= 0).all()
