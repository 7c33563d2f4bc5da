#!/bin/bash
# rebuild stats.cu with -G (device debug) into the library, then run the failing test under memcheck
set -x
cd /root/repo
python __graft_entry__.py build > gpurun_out/build.log 2>&1
EXTRA_G=1 python - <<'PY'
import os, subprocess, sys
sys.path.insert(0, ".")
from paper_2103_14409_b200 import build as B
src = os.path.join(B.CSRC, "stats.cu")
obj = os.path.join(B.BUILD, "stats.cu.o")
cmd = [B.NVCC] + [f for f in B.flags() if f != "-lineinfo"] + ["-G", "--fmad=false", "-c", src, "-o", obj]
print(subprocess.run(cmd, capture_output=True, text=True).stderr[-2000:])
os.utime(obj)
B.build()
PY
LSCAT_SEL_DEBUG=1 timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_reduce.py -k "wide" -x -q > gpurun_out/san_wideG.log 2>&1
grep -E "^sel" gpurun_out/san_wideG.log | head -20
grep -A4 "^========= Invalid" gpurun_out/san_wideG.log | grep -E "Invalid|at |Access" | sed "s/by thread.*//" | sort | uniq -c | sort -rn | head -8
tail -3 gpurun_out/san_wideG.log
