"""configs[4] at 10^9 rows: reduce + stats a few times (ncu launch lists / timing of the large-table
selection).  argv: reps [n_rows]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000_000
c = L.Ctx(0, seed=0x15CA7)
tab = c.gen_table(n, n // 256, preset=L.PRESET_T4, seed=10 ** 9, offsets=False)
o = L.reduce_opts(32, 8)
s = torch.cuda.current_stream()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for i in range(reps):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(s)
    c.reduce_table(tab, o, per_group=False)
    e1.record(s)
    st = c.stats(o, percentiles=PCTS)
    e2.record(s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {i}: reduce {e0.elapsed_time(e1)*1e3:.1f} us, stats {e1.elapsed_time(e2)*1e3:.1f} us, "
          f"host total {1e6*(t2-t0):.1f} us")
print("pct_perf", st["pct_perf"])
