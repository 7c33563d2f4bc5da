"""Table rows/s of reduce + stats with the percentiles in the reduce options (R-27) against
the usual two-call path, configs[2]-[4] on one GPU (cold L2 per rep, median of 10)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
c = L.Ctx(0, seed=0x15CA7)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
out = {}
for name, n, K, preset, seed, offs in (("gtx980", 2_140_796, 8363, L.PRESET_GTX980, 980, True),
                                       ("t4", 5_028_536, 19_683, L.PRESET_T4, 4, True),
                                       ("scaled_1e9", 1_000_000_000, 3_906_250, L.PRESET_T4, 10 ** 9, False)):
    if os.environ.get("LSCAT_TABLE_SMALL_ONLY") and n > 10 ** 8 or (os.environ.get("LSCAT_TABLE_ONE") and n > 3_000_000):
        continue
    tab = c.gen_table(n, K, preset=preset, seed=seed, offsets=offs)
    res = {}
    for mode in ("usual", "early"):
        kw = {} if mode == "usual" else dict(percentiles=PCTS)
        o = L.reduce_opts(32, 8, **kw)
        for _ in range(3):
            c.reduce_table(tab, o, per_group=False)
            st = c.stats(o, percentiles=PCTS)
        ts, rs = [], []
        for _ in range(10):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            flush.zero_()
            torch.cuda.synchronize()
            e0.record(s)
            c.reduce_table(tab, o, per_group=False)
            e1.record(s)
            st = c.stats(o, percentiles=PCTS)
            e2.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e2))
            rs.append(e0.elapsed_time(e1))
        res[mode] = {"ms": round(statistics.median(ts), 4), "ms_reduce_call": round(statistics.median(rs), 4),
                     "pct_perf": st["pct_perf"], "pct_gain": st["pct_gain"]}
        print(name, mode, res[mode]["ms"], file=sys.stderr, flush=True)
    res["same_values"] = all(res[m]["pct_perf"] == res["usual"]["pct_perf"] and
                             res[m]["pct_gain"] == res["usual"]["pct_gain"] for m in res if m != "usual")
    out[name] = res
    del tab
    torch.cuda.empty_cache()
print(json.dumps(out))
