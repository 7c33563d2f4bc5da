"""compute-sanitizer target for the session-3 changes: the one-launch small-table selection
(staged histograms, warp target path, radix select of bins above 128 keys; configs[2] shape)
with the partials' side-branch copy, the general (> 32 targets) path, and a GLOBALTIMER sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
c = L.Ctx(0)
tab = c.gen_table(2_140_796, 8363, preset=L.PRESET_GTX980, seed=980)
o = L.reduce_opts(32, 8, percentiles=PCTS)
for _ in range(3):  # direct, then captured, then replayed
    c.reduce_table(tab, o, per_group=False)
    st = c.stats(o, percentiles=PCTS)
many = list(np.linspace(0.0, 1.0, 40))
o2 = L.reduce_opts(32, 8, percentiles=many)
c.reduce_table(tab, o2, per_group=False)
st2 = c.stats(o2, percentiles=many)
c.register_suite([L.K_EUCLID], [256])
c.sweep([L.K_EUCLID], [256], [64, 256], warmup=1, brackets=3, launches=4, timer=L.TIMER_GLOBALTIMER)
torch.cuda.synchronize()
print("ok", st["pct_perf"][4], st2["pct_perf"][20])
