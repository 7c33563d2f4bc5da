#!/bin/bash
# transpose calibration (round 1): experimental switches (TP_TMA with kern_tp_tma.cu, TP_PERM, TP_PERM_TMA)
# measured and removed (results: profiles/r01_summary.md)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
{
timeout 120 python scripts/suite_probe.py transpose 8192
timeout 120 python scripts/suite_probe.py transpose 4096
rm -f paper_2103_14409_b200/_build/kern_move.cu.o
LSCAT_NVCC_EXTRA="-DTP_TMA=1" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null
echo "variant TP_TMA=1"
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sweep.py -q -x -k "transpose or data_movement or pdl" 2>&1 | tail -1
timeout 120 python scripts/suite_probe.py transpose 8192
timeout 120 python scripts/suite_probe.py transpose 4096
} > gpurun_out/tp_tma.jsonl 2>&1
rm -f paper_2103_14409_b200/_build/kern_move.cu.o
echo done
