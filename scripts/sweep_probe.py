"""Per-N mean/min/max per-launch time of a PDL-graph sweep of one kernel over all 32 blocks
(the bench's launch path, shorter brackets):  python scripts/sweep_probe.py KERNEL N1,N2,..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

name, sizes = sys.argv[1], [int(x) for x in sys.argv[2].split(",")]
k = L.KERNELS[name]
c = L.Ctx(0)
c.register_suite([k], sizes)
blocks = list(range(32, 1025, 32))
c.sweep([k], sizes, blocks, warmup=1, brackets=2, launches=100, launch_mode=L.LAUNCH_GRAPH_PDL)
t = c.sweep([k], sizes, blocks, warmup=1, brackets=3, launches=500,
            launch_mode=L.LAUNCH_GRAPH_PDL).to_numpy()
out = {"kernel": name, "env": {k2: v for k2, v in os.environ.items() if k2.startswith("LSCAT_")}}
for gi, n in enumerate(sizes):
    a, b = t["group_offset"][gi], t["group_offset"][gi + 1]
    us = t["runtime_ms"][a:b] * 1e3
    nbytes, _ = L.kernel_work(k, n)
    out[str(n)] = {"mean": round(float(us.mean()), 3), "min": round(float(us.min()), 3),
                   "max": round(float(us.max()), 3), "best_gbs": round(float(nbytes / (us.min() * 1e-6) / 1e9), 1),
                   "by_block": [round(float(x), 2) for x in us]}
print(json.dumps(out))
