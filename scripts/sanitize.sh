#!/bin/bash
# compute-sanitizer over scripts/sanitize_run.py (memcheck, racecheck, synccheck)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.log
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py --gemm-multi > gpurun_out/sanitize_memcheck_gemm.log 2>&1
echo "memcheck (+ persistent GEMM multi-tile) rc=$?"; tail -2 gpurun_out/sanitize_memcheck_gemm.log
