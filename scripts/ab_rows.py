"""A/B of the row kernels in one box session: per-block per-launch time of euclid at N = 4096
and 8192 (plain graph brackets, warm L2 as in the bench table, and cold L2), loading the
library given on the command line (the current build or an older build kept for comparison).

    python scripts/ab_rows.py paper_2103_14409_b200/liblscat.so [tag]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2103_14409_b200 import lscat  # noqa: E402

lib = sys.argv[1]
tag = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(lib)
lscat.load(lib)
import paper_2103_14409_b200 as L  # noqa: E402

c = L.Ctx(0, seed=0x15CA7)
blocks = list(range(32, 1025, 32))
sizes = [4096, 8192]
c.register_suite([L.K_EUCLID], sizes)
out = {"tag": tag}
for mode, l2 in (("warm", L.L2_WARM), ("cold", L.L2_ROTATE)):
    c.sweep([L.K_EUCLID], sizes, blocks, warmup=1, brackets=3, launches=50, l2_mode=l2)
    t = c.sweep([L.K_EUCLID], sizes, blocks, warmup=1, brackets=5, launches=200, l2_mode=l2).to_numpy()
    rt = t["runtime_ms"] * 1e3
    for i, n in enumerate(sizes):
        v = rt[i * 32:(i + 1) * 32]
        out[f"{mode}_{n}"] = {"min": round(float(v.min()), 2), "mean": round(float(v.mean()), 2),
                              "max": round(float(v.max()), 2)}
        if os.environ.get("AB_BY_BLOCK"):
            out[f"{mode}_{n}"]["by_block"] = [round(float(x), 2) for x in v]
print(json.dumps(out))
