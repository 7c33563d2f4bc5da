#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for tw in auto 1 2 4 8; do
  if [ $tw = auto ]; then timeout 300 python scripts/sweep_probe.py euclid 64,256,512,1024,2048;
  else LSCAT_ROW_TEAM_WARPS=$tw timeout 300 python scripts/sweep_probe.py euclid 64,256,512,1024,2048; fi
done > gpurun_out/tw_probe.jsonl 2>&1
echo done
