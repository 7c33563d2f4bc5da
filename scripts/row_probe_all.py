"""euclid per-launch time at every block size (CUDA events, 100 launches), N from env."""
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
for b in range(32, 1025, 32):
    for _ in range(10):
        c.launch(L.K_EUCLID, n, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(100):
        c.launch(L.K_EUCLID, n, b)
    e1.record()
    torch.cuda.synchronize()
    res[b] = round(e0.elapsed_time(e1) / 100 * 1e3, 1)
v = sorted(res.values())
print(json.dumps({"N": n, "median": v[len(v) // 2], "max": v[-1], "us": res}))
