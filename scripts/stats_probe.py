"""Time reduce_table and stats (no percentiles / 9 percentiles) on the BASELINE table
configs (device-resident), CUDA events on the current stream, median of 20."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
c = L.Ctx(0)
s = torch.cuda.current_stream()
cases = [("gtx980", dict(n_rows_global=2_140_796, n_kernels=8363, preset=L.PRESET_GTX980, seed=980)),
         ("t4", dict(n_rows_global=5_028_536, n_kernels=19_683, preset=L.PRESET_T4, seed=4)),
         ("1e9", dict(n_rows_global=1_000_000_000, n_kernels=3_906_250, preset=L.PRESET_T4, seed=10 ** 9,
                      offsets=False))]
for name, kw in cases:
    tab = c.gen_table(**kw)
    o = L.reduce_opts(32, 8)
    res = {}
    for label, pcts in (("none", []), ("p9", PCTS)):
        tr, ts, tw = [], [], []
        for i in range(23):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            torch.cuda.synchronize()
            e0.record(s)
            c.reduce_table(tab, o, per_group=False)
            e1.record(s)
            w0 = time.perf_counter()
            c.stats(o, percentiles=pcts)
            w1 = time.perf_counter()
            e2.record(s)
            torch.cuda.synchronize()
            if i >= 3:
                tr.append(e0.elapsed_time(e1) * 1e3)
                ts.append(e1.elapsed_time(e2) * 1e3)
                tw.append((w1 - w0) * 1e6)
        res[label] = {"reduce_us": round(statistics.median(tr), 1), "stats_us": round(statistics.median(ts), 1),
                      "stats_host_wall_us": round(statistics.median(tw), 1)}
    print(json.dumps({"table": name, **res}))
    del tab
    torch.cuda.empty_cache()
