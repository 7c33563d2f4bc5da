"""Small end-to-end exercise of every kernel of liblscat for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck), e.g.

    compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py

Sizes are tiny (ragged tails included) so the instrumented run finishes in seconds.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

skip_gemm = "--no-gemm" in sys.argv
c = L.Ctx(0)
ks = [L.K_EUCLID, L.K_MATVEC, L.K_TRANSPOSE, L.K_AXPY, L.K_ROWSUM, L.K_COLSUM, L.K_STENCIL5]
if not skip_gemm:
    ks.append(L.K_GEMM_BF16)
ns = [64, 136]
bs = [32, 96, 128, 256, 1024]
c.register_suite(ks, ns)
tab = c.sweep(ks, ns, bs, warmup=1, brackets=2, launches=2)
# PDL graph brackets (griddepcontrol) and a size where the warp-unit loops iterate
ks32 = [k for k in ks if k != L.K_GEMM_BF16]
c.register_suite(ks32, [1040])
c.sweep(ks32, [1040], [32, 160, 1024], warmup=1, brackets=2, launches=3, launch_mode=L.LAUNCH_GRAPH_PDL)
o = L.reduce_opts(len(bs), len(ns), block_profile=1)
c.reduce_table(tab, o)
st = c.stats(o, percentiles=[0.1, 0.5, 0.9])
# ragged / uniform / point-sharded-shaped generated tables
for kw in (dict(n_rows_global=50_000, n_kernels=200, preset=0, seed=1),
           dict(n_rows_global=32 * 3000, n_kernels=375, preset=1, seed=2, offsets=False),
           dict(n_rows_global=40_000, n_kernels=100, preset=0, seed=3, block_mod=3, block_rem=2)):
    t = c.gen_table(**kw)
    o32 = L.reduce_opts(32, 8, block_profile=1)
    c.reduce_table(t, o32)
    c.stats(o32, percentiles=[0.01, 0.5, 0.99])
# ingest, aggregation experiment, side analyses
h = c.gen_table(20_000, 100, preset=0, seed=4).to_numpy()
p = np.random.default_rng(0).permutation(h["n_rows"])
gk = np.repeat(h["group_kernel"], np.diff(h["group_offset"]))[p]
gm = np.repeat(h["group_matrix"], np.diff(h["group_offset"]))[p]
T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()
c.ingest(T(gk.astype(np.uint32), np.int32), T(gm.astype(np.uint32), np.int32),
         T(h["block_id"][p], np.int16), T(h["runtime_ms"][p], np.float32))
c.aggregation_experiment(torch.rand(1000, device="cuda") + 1, k=10, reps=200, seed=1)
c.occupancy_block(L.K_EUCLID, list(range(32, 1025, 32)))
c.timeout_curve(tab, [1e-3, 1.0], 1, 2, 2)
if "--round2" in sys.argv:  # round-2 paths: early selection, graph replay, sampled pass, roll-up
    P9 = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
    small = c.gen_table(200_000, 800, preset=0, seed=5)
    oe = L.reduce_opts(32, 8, percentiles=P9, kernel_rollup=1)
    for _ in range(3):  # the third call replays the captured graph
        c.reduce_table(small, oe, per_group=False)
        c.stats(oe, percentiles=P9)
    big = c.gen_table(32 * (1 << 20) + 32 * 4096, (1 << 20) // 8 + 512, preset=0, seed=6, offsets=False)
    ob = L.reduce_opts(32, 8, percentiles=P9, kernel_rollup=1)
    c.reduce_table(big, ob, per_group=False)  # > 2^20 groups: sampled selection + sel_finish
    c.stats(ob, percentiles=P9)
    c.stats(ob, percentiles=[0.3, 0.6])  # another list: the usual selection
if "--gemm-multi" in sys.argv:  # persistent GEMM with two tiles per CTA (153 tiles)
    c.register_suite([L.K_GEMM_BF16], [2056])
    for b in (192, 256):
        c.launch(L.K_GEMM_BF16, 2056, b)
torch.cuda.synchronize()
print("sanitize run ok", st["n_rows"], c.launch_count())
