"""Worker for tests/test_gpu_nccl.py (launched by torchrun, one process per GPU): the a9 merge
over the real NCCL transport.  Each rank holds a point-sharded slice (rows of block ids
b % world == rank) of the T4-scale table, reduces it with the per-group NCCL MIN/MAX/SUM merge
and computes the stats (collective); rank 0 compares with the oracle on the whole table."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

PCTS = [0.01, 0.1, 0.5, 0.9, 0.99]


def main():
    rank, world, lrank = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lrank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    uid = [L.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ctx = L.Ctx(lrank)
    ctx.comm_init(uid[0], rank, world)
    n, K = 5_028_536, 19_683
    tab = ctx.gen_table(n, K, preset=L.PRESET_T4, seed=4, block_mod=world, block_rem=rank)
    o = L.reduce_opts(32, 8, point_sharded=1)
    ctx.reduce_table(tab, o, per_group=False)
    st = ctx.stats(o, percentiles=PCTS)
    objs = [None] * world
    dist.all_gather_object(objs, {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in st.items()})
    ok = True
    if rank == 0:
        import numpy as np
        from oracle import table as OT
        from synth import gen_table
        h = gen_table(n, K, preset="t4", seed=4)
        ref = OT.reduce_table(h["runtime_ms"], h["block_id"], h["group_offset"],
                              group_matrix=h["group_matrix"], percentiles=PCTS)
        for r, s in enumerate(objs):
            for k, v in ref.counters.items():
                if s[k] != v:
                    print(f"rank {r}: {k} {s[k]} != {v}")
                    ok = False
            if list(s["pct_perf"]) != list(ref.percentiles["perf"]) or list(s["pct_gain"]) != list(ref.percentiles["gain"]):
                print(f"rank {r}: percentiles differ")
                ok = False
            if not (np.asarray(s["best_block_hist"]) == ref.best_block_hist).all():
                print(f"rank {r}: best_block_hist differs")
                ok = False
        print("nccl merge", "ok" if ok else "FAILED", "world", world)
    ok_t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
    ctx.close()
    dist.destroy_process_group()
    sys.exit(0 if ok_t.item() == 1 else 1)


if __name__ == "__main__":
    main()
