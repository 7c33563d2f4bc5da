#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_sweep.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_sweep.log
for m in graph_pdl graph; do
  timeout 900 python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu --no-e2e --launch $m > gpurun_out/bench_$m.log 2>&1; echo "bench $m rc=$?"
done
