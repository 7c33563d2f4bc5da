#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sweep.py -x -q > gpurun_out/pytest_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -3 gpurun_out/pytest_kernels.log
{
for k in stencil5 euclid matvec rowsum; do timeout 120 python scripts/suite_probe.py $k 8192; done
for k in stencil5 euclid; do timeout 120 python scripts/suite_probe.py $k 4096; done
} > gpurun_out/probe3.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:transpose -c 1 -s 1 -o gpurun_out/prof_transpose -f python scripts/profile_kernels.py kernel transpose 8192 256 > gpurun_out/ncu_tp.log 2>&1; echo "ncu rc=$?"
echo done
