#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
python __graft_entry__.py build > gpurun_out/s3/build.log 2>&1 || exit 1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_small.py > gpurun_out/s3/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/s3/sanitize_$tool.log
done
