"""configs[4] (10^9 rows) reduce with and without the kernel roll-up (ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

c = L.Ctx(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
tab = c.gen_table(n, n // 256, preset=L.PRESET_T4, seed=10 ** 9, offsets=False)
for roll in (0, 1, 0, 1):
    o = L.reduce_opts(32, 8, kernel_rollup=roll)
    c.reduce_table(tab, o, per_group=False)
    c.stats(o, percentiles=[0.5])
torch.cuda.synchronize()
print("ok")
