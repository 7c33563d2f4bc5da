#!/bin/bash
# transpose calibration (round 1): experimental switches (TP_TMA with kern_tp_tma.cu, TP_PERM, TP_PERM_TMA)
# measured and removed (results: profiles/r01_summary.md)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
{
for v in "TP_PERM=1" "TP_TMA=1 -DTP_PERM_TMA"; do
  rm -f paper_2103_14409_b200/_build/kern_move.cu.o paper_2103_14409_b200/_build/kern_tp_tma.cu.o
  LSCAT_NVCC_EXTRA="-D$v" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null
  echo "variant $v"
  timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "transpose or data_movement" 2>&1 | tail -1
  timeout 120 python scripts/suite_probe.py transpose 8192
  timeout 120 python scripts/suite_probe.py transpose 4096
done
} > gpurun_out/tp_perm.jsonl 2>&1
rm -f paper_2103_14409_b200/_build/kern_move.cu.o paper_2103_14409_b200/_build/kern_tp_tma.cu.o
echo done
