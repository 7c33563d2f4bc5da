#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
{
timeout 300 python scripts/sweep_probe.py euclid 4096,8192
LSCAT_ROW_L2PERSIST=1 timeout 300 python scripts/sweep_probe.py euclid 4096,8192
} > gpurun_out/l2persist.jsonl 2>&1
echo done
