#!/bin/bash
# transpose variants (tiles per warp unit, orientation, register budget) + probes of the
# reworked stencil/row kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -3 gpurun_out/pytest_kernels.log
{
for k in stencil5 euclid; do timeout 120 python scripts/suite_probe.py $k 8192; done
for v in "TP_TPW=2 -DTP_VERT=1 -DTP_MINB_THREADS=768" "TP_TPW=4 -DTP_VERT=1 -DTP_MINB_THREADS=512" "TP_TPW=1 -DTP_MINB_THREADS=2048"; do
  rm -f paper_2103_14409_b200/_build/kern_move.cu.o
  LSCAT_NVCC_EXTRA="-D$v" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null || { echo "build failed $v"; continue; }
  echo "variant $v"
  timeout 120 python scripts/suite_probe.py transpose 8192
done
} > gpurun_out/tp_variants.jsonl 2>&1
rm -f paper_2103_14409_b200/_build/kern_move.cu.o
echo done
