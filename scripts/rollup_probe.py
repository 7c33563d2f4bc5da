"""configs[4] (10^9 rows) reduce (with / without the kernel roll-up) + 9 percentiles, for ncu
launch lists:  python scripts/rollup_probe.py [n_rows] [roll-up flags, e.g. 0,1,0,1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

c = L.Ctx(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
tab = c.gen_table(n, n // 256, preset=L.PRESET_T4, seed=10 ** 9, offsets=False)
PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
rolls = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 0, 1]
for roll in rolls:
    o = L.reduce_opts(32, 8, kernel_rollup=roll)
    c.reduce_table(tab, o, per_group=False)
    c.stats(o, percentiles=PCTS)
torch.cuda.synchronize()
print("ok")
