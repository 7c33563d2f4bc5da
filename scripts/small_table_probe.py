"""configs[2] reduce + stats, a few times (ncu launch lists / timing of the small-table path)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
c = L.Ctx(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_140_796
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
tab = c.gen_table(n, 8363 if n < 3_000_000 else 19_683, preset=L.PRESET_GTX980, seed=980)
o = L.reduce_opts(32, 8)
s = torch.cuda.current_stream()
for i in range(reps):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(s)
    c.reduce_table(tab, o, per_group=False)
    e1.record(s)
    t1 = time.perf_counter()
    c.stats(o, percentiles=PCTS)
    e2.record(s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {i}: reduce {e0.elapsed_time(e1)*1e3:.1f} us (host {1e6*(t1-t0):.1f}), "
          f"stats {e1.elapsed_time(e2)*1e3:.1f} us (host {1e6*(t2-t1):.1f})")
