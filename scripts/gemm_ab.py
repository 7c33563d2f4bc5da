"""A/B of GEMM block configurations at N = 8192 in the burst regime (power state matters:
the B200 throttles under sustained tensor load): interleaved short bursts after idle gaps."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

n = 8192
blocks = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128,256").split(",")]
c = L.Ctx(0)
c.register_suite([L.K_GEMM_BF16], [n])
res = {b: [] for b in blocks}
for b in blocks:
    c.launch(L.K_GEMM_BF16, n, b)
torch.cuda.synchronize()
for rep in range(12):
    for b in blocks:
        time.sleep(0.25)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            c.launch(L.K_GEMM_BF16, n, b)
        e1.record()
        torch.cuda.synchronize()
        res[b].append(e0.elapsed_time(e1) / 5 * 1e3)
flops = 2 * n ** 3
print(json.dumps({str(b): {"median_us": round(statistics.median(v), 1), "min_us": round(min(v), 1),
                           "tflops_median": round(flops / (statistics.median(v) * 1e-6) / 1e12, 1)}
                  for b, v in res.items()}))
