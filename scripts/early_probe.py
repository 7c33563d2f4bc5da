"""The 10^9-row table with the percentiles in the reduce options (R-27): a few reduce + stats
calls (ncu launch-list target; LSCAT_SEL_DEBUG=1 prints the fused plan and sel_finish phases)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
keep = int(sys.argv[3]) if len(sys.argv) > 3 else 1
c = L.Ctx(0, seed=0x15CA7)
tab = c.gen_table(n, n // 256, preset=L.PRESET_T4, seed=10 ** 9, offsets=False)
o = L.reduce_opts(32, 8, percentiles=PCTS, keep_values=keep)
s = torch.cuda.current_stream()
for i in range(reps):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    e0.record(s)
    c.reduce_table(tab, o, per_group=False)
    e1.record(s)
    st = c.stats(o, percentiles=PCTS)
    e2.record(s)
    torch.cuda.synchronize()
    print(f"rep {i}: reduce call {e0.elapsed_time(e1):.3f} ms, total {e0.elapsed_time(e2):.3f} ms", flush=True)
print(st["pct_perf"], st["pct_gain"])
