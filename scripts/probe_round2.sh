#!/bin/bash
# kernel parity tests + per-block probes of the reworked suite kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sweep.py -x -q > gpurun_out/pytest_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -3 gpurun_out/pytest_kernels.log
{
for k in transpose stencil5 colsum euclid matvec rowsum axpy; do timeout 120 python scripts/suite_probe.py $k 8192; done
for k in transpose stencil5 colsum; do timeout 120 python scripts/suite_probe.py $k 4096; done
for n in 2048 1024 512 256; do
  for tw in auto 1 2 4; do
    if [ $tw = auto ]; then timeout 120 python scripts/suite_probe.py euclid $n; else LSCAT_ROW_TEAM_WARPS=$tw timeout 120 python scripts/suite_probe.py euclid $n; fi
  done
done
timeout 120 python scripts/suite_probe.py euclid 4096
} > gpurun_out/probe2.jsonl 2>&1
echo probes done
