"""Time euclid at N=8192 for several blocks (CUDA events, 200 launches) - used with the
LSCAT_ROW_TEAM_WARPS override to calibrate the row-kernel team heuristic."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

c = L.Ctx(0)
n = int(os.environ.get("N", "8192"))
c.register_suite([L.K_EUCLID], [n])
res = {}
for b in [32, 64, 96, 128, 256, 512, 800, 1024]:
    for _ in range(20):
        c.launch(L.K_EUCLID, n, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(200):
        c.launch(L.K_EUCLID, n, b)
    e1.record()
    torch.cuda.synchronize()
    res[b] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
print(json.dumps({"tw": os.environ.get("LSCAT_ROW_TEAM_WARPS", "auto"), "N": n, "us": res}))
