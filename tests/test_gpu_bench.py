"""bench.py end to end at the tiny policy (the driver runs it at the paper policy at round end):
one JSON line with the contract's keys, a cold roofline in a plausible range, the CPU baseline
with the host record, e2e byte counts, and the secondaries (tables incl. 10^9 rows, the full
suite, the launch-mode comparison, the cold suite roofline, the occupancy-API comparison)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_tiny_policy_json():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    r = subprocess.run([sys.executable, "bench.py", "--policy", "tiny", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "clocks", "gpu_launches", "roofline",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["gpu_launches"] > 0
    roof = d["roofline"]
    assert roof["bound"] == "hbm" and 0.3 < roof["frac"] < 1.25, roof
    assert roof["traffic"] and roof["achieved"] > 0
    cpu = d["cpu_baseline"]
    assert cpu["kind"] == "oracle" and cpu["cores"] >= 1 and cpu["host"]["nproc"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    sec = d["secondary"]
    for k in ("tables", "full_suite_fast_policy", "launch_modes", "suite_roofline_n8192", "occupancy_api"):
        assert k in sec, k
    assert sec["tables"]["scaled_1e9"]["check_n_rows"] == 1_000_000_000
    assert sec["full_suite_fast_policy"]["points"] == 2048
    assert set(sec["occupancy_api"]) >= {"euclid", "gemm_bf16"}
