"""Per-launch time of one suite kernel at every block size (CUDA events, 100 launches after
10 warm-up launches):  python scripts/suite_probe.py KERNEL N   (KERNEL: euclid, transpose, ...)
Env LSCAT_ROW_TEAM_WARPS overrides the row kernels' team size (calibration)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
k = L.KERNELS[name]
c = L.Ctx(0)
c.register_suite([k], [n])
nbytes, flops = L.kernel_work(k, n)
res = {}
for b in range(32, 1025, 32):
    try:
        for _ in range(10):
            c.launch(k, n, b)
    except Exception:
        continue
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(100):
        c.launch(k, n, b)
    e1.record()
    torch.cuda.synchronize()
    res[b] = round(e0.elapsed_time(e1) / 100 * 1e3, 2)
v = sorted(res.values())
best = min(res, key=res.get)
print(json.dumps({"kernel": name, "N": n, "tw": os.environ.get("LSCAT_ROW_TEAM_WARPS", "auto"),
                  "mean": round(sum(v) / len(v), 2), "median": v[len(v) // 2], "max": v[-1],
                  "best_block": best, "best_gbs": round(nbytes / (res[best] * 1e-6) / 1e9, 1),
                  "us": res}))
