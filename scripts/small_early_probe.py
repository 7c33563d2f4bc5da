"""configs[2] / configs[3] reduce + 9 percentiles with the percentiles in the reduce options
(R-27: sel_small enqueued behind the reducer, graph replay), a few reps: the target of the ncu
captures of reduce_groups_kernel / sel_small (round 2, session 3)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
c = L.Ctx(0)
which = sys.argv[1] if len(sys.argv) > 1 else "gtx980"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if which == "gtx980":
    tab = c.gen_table(2_140_796, 8363, preset=L.PRESET_GTX980, seed=980)
else:
    tab = c.gen_table(5_028_536, 19_683, preset=L.PRESET_T4, seed=4)
rollup = int(sys.argv[3]) if len(sys.argv) > 3 else 0
o = L.reduce_opts(32, 8, percentiles=PCTS, kernel_rollup=rollup)
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
    t1 = time.perf_counter()
    st = c.stats(o, percentiles=PCTS)
    e2.record(s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {i}: reduce {e0.elapsed_time(e1)*1e3:.1f} us (host {1e6*(t1-t0):.1f}), "
          f"stats {e1.elapsed_time(e2)*1e3:.1f} us (host {1e6*(t2-t1):.1f}) total {e0.elapsed_time(e2)*1e3:.1f}")
print("pct_perf", st["pct_perf"])
