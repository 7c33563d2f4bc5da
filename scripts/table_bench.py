"""bench.py's table rows/s secondary alone (configs[2]-[4], one GPU): reduce + stats timings."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_14409_b200 as L  # noqa: E402

c = L.Ctx(0, seed=0x15CA7)
hbm = bench.load_peaks()[0]
out = bench.table_benches(c, L, hbm, 0, 1, torch.cuda.synchronize, lambda x: x, cpu_rows=False)
print(json.dumps(out))
