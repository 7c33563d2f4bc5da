"""a9 over the real NCCL transport: 2 ranks on 2 GPUs (torchrun), point-sharded T4-scale table,
bit-exact against the oracle on every rank; and bench.py's multi-rank path (tiny policy).
Skipped on a box with fewer than 2 GPUs (this round's boxes have one; the local-transport
tests in test_gpu_multirank.py run the same merge code on one GPU)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _need_two_gpus():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")


def _torchrun(args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533"] + args
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)


def test_nccl_point_sharded_merge_two_ranks():
    _need_two_gpus()
    r = _torchrun([os.path.join(ROOT, "tests", "nccl_worker.py")])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "nccl merge ok" in r.stdout


def test_bench_two_ranks_tiny_policy():
    _need_two_gpus()
    r = _torchrun([os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1",
                   "--policy", "tiny"])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    import json
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["stats_last_step"]["n_rows"] == 256
