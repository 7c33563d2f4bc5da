"""Per-launch time of the test-only spin kernel with spin_ns = 0 (an almost empty kernel) in the
sweep's launch modes, beside euclid at N = 64 / 256: the launch floor the small-N points sit on."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_14409_b200 as L  # noqa: E402

c = L.Ctx(0)
c.register_suite([L.K_EUCLID], [64, 256])
out = {}
for name, mode in (("graph", L.LAUNCH_GRAPH), ("graph_pdl", L.LAUNCH_GRAPH_PDL), ("stream", L.LAUNCH_STREAM)):
    t = c.sweep([L.K_SPIN], [1], [32, 256, 1024], warmup=1, brackets=5, launches=1000, spin_ns=0,
                launch_mode=mode).to_numpy()
    e = c.sweep([L.K_EUCLID], [64, 256], [32, 256, 1024], warmup=1, brackets=5, launches=1000,
                launch_mode=mode).to_numpy()
    out[name] = {"empty_us": [round(float(x) * 1e3, 3) for x in t["runtime_ms"]],
                 "euclid_64_256_us": [round(float(x) * 1e3, 3) for x in e["runtime_ms"]]}
print(json.dumps(out))
