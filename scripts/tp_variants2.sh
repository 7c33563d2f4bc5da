#!/bin/bash
# transpose calibration (round 1): the -D variants (TP_STORE_PLAIN, TP_ORDER, TP_COPY, TP_PIPE) were
# experimental switches measured and then removed from kern_move.cu (results: profiles/r01_summary.md)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "transpose or data_movement" 2>&1 | tail -1
{
timeout 120 python scripts/suite_probe.py transpose 8192
for v in "TP_PIPE=0" "TP_PIPE_MINB_THREADS=768" "TP_PIPE_MINB_THREADS=512"; do
  rm -f paper_2103_14409_b200/_build/kern_move.cu.o
  LSCAT_NVCC_EXTRA="-D$v" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null || { echo "build failed $v"; continue; }
  echo "variant $v"
  timeout 120 python scripts/suite_probe.py transpose 8192
done
} > gpurun_out/tp_variants2.jsonl 2>&1
rm -f paper_2103_14409_b200/_build/kern_move.cu.o
echo done
