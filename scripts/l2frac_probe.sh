#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "vector or euclid" 2>&1 | tail -1
for f in 0 0.3 0.45 0.6 0.75; do LSCAT_ROW_L2FRAC=$f timeout 300 python scripts/sweep_probe.py euclid 4096,8192; done > gpurun_out/l2frac.jsonl 2>&1
echo done
