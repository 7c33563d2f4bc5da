#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "vector or euclid" > gpurun_out/pytest_k.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_k.log
for v in 0 1; do LSCAT_ROW_L2KEEP=$v timeout 300 python scripts/sweep_probe.py euclid 512,1024,2048,4096,8192; done > gpurun_out/l2keep.jsonl 2>&1
timeout 300 python scripts/sweep_probe.py euclid 512,1024,2048,4096,8192 >> gpurun_out/l2keep.jsonl 2>&1
echo done
