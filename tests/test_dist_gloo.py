"""World-size-2 CPU tests (gloo) of the multi-GPU host logic:

* the planner: every rank computes the same LPT partition independently; union = all points;
* group-aligned table shards: per-rank oracle partials SUM-merged over the process group equal
  the single-table result (the a9 partial-vector merge);
* point-sharded tables: per-group MIN(argmin key) / MAX(largest-block code) / SUM(counts)
  merged over the group reproduce the full table's per-group argmin and counts.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _plan_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    from paper_2103_14409_b200 import lscat
    ks = [lscat.K_EUCLID, lscat.K_GEMM_BF16, lscat.K_AXPY]
    sizes = [64, 256, 1024, 4096, 8192]
    blocks = list(range(32, 1025, 32))
    mine = lscat.plan(ks, sizes, blocks, rank, world)
    theirs = lscat.plan(ks, sizes, blocks, 1 - rank, world)
    objs = [None, None]
    dist.all_gather_object(objs, (mine.tolist(), theirs.tolist()))
    ok = objs[0][0] == objs[1][1] and objs[1][0] == objs[0][1]
    allp = sorted(objs[0][0] + objs[1][0])
    ok = ok and allp == list(range(len(ks) * len(sizes) * len(blocks)))
    q.put((rank, ok))
    dist.destroy_process_group()


def _merge_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    from oracle import table as OT
    from synth import gen_table
    n, K = 120_000, 400
    full = gen_table(n, K, preset="t4", seed=21)
    G = full["n_groups"]
    ref = OT.reduce_table(full["runtime_ms"], full["block_id"], full["group_offset"],
                          group_matrix=full["group_matrix"])
    ok = True
    # -- group-aligned shards: SUM of integer partials
    g0, g1 = G * rank // world, G * (rank + 1) // world
    s = gen_table(n, K, preset="t4", seed=21, group_begin=g0, group_end=g1)
    part = OT.reduce_table(s["runtime_ms"], s["block_id"], s["group_offset"],
                           group_matrix=s["group_matrix"])
    vec = torch.tensor([part.counters[k] for k in OT.COUNTERS] + part.perf_hist.tolist()
                       + part.gain_hist.tolist() + part.best_block_hist.ravel().tolist(),
                       dtype=torch.int64)
    dist.all_reduce(vec, op=dist.ReduceOp.SUM)
    want = torch.tensor([ref.counters[k] for k in OT.COUNTERS] + ref.perf_hist.tolist()
                        + ref.gain_hist.tolist() + ref.best_block_hist.ravel().tolist(),
                        dtype=torch.int64)
    ok = ok and torch.equal(vec, want)
    # -- point-sharded: rows with block_id % world == rank
    p = gen_table(n, K, preset="t4", seed=21, block_mod=world, block_rem=rank)
    off, rt, bid = p["group_offset"], p["runtime_ms"], p["block_id"].astype(np.int64)
    key = np.full(G, np.iinfo(np.int64).max, np.int64)
    lcode = np.zeros(G, np.int64)
    cnt = np.zeros((G, 3), np.int64)
    bits = rt.view(np.uint32).astype(np.int64)
    okr = np.isfinite(rt) & (rt > 0)
    for g in range(G):
        r = slice(off[g], off[g + 1])
        o = okr[r]
        if o.any():
            key[g] = ((bits[r][o] << 32) | bid[r][o]).min()
        li = np.nonzero(bid[r] == 31)[0]
        if li.size:
            lcode[g] = ((1 << 32) | bits[r][li[0]]) if o[li[0]] else 1
        cnt[g] = (o.sum(), np.isnan(rt[r]).sum(), off[g + 1] - off[g])
    K_, L_, C_ = torch.from_numpy(key), torch.from_numpy(lcode), torch.from_numpy(cnt)
    dist.all_reduce(K_, op=dist.ReduceOp.MIN)
    dist.all_reduce(L_, op=dist.ReduceOp.MAX)
    dist.all_reduce(C_, op=dist.ReduceOp.SUM)
    best = np.where(K_.numpy() == np.iinfo(np.int64).max, 0xFFFF, K_.numpy() & 0xFFFF)
    ok = ok and (best == ref.best_block).all()
    ok = ok and int(C_[:, 0].sum()) == ref.counters["n_ok"]
    ok = ok and int(C_[:, 2].sum()) == ref.counters["n_rows"]
    rd = (L_.numpy() >> 32) == 1
    ok = ok and int((rd & (K_.numpy() != np.iinfo(np.int64).max)).sum()) == ref.counters["n_ratio_defined"]
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("worker", [_plan_worker, _merge_worker])
def test_world2_gloo(worker):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.start_processes(worker, args=(2, port, q), nprocs=2, join=True, start_method="spawn")
    res = sorted(q.get() for _ in range(2))
    assert res == [(0, True), (1, True)]
