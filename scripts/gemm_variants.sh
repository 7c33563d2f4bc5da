#!/bin/bash
# CTA-pair GEMM pipeline depth (GEMM2_STAGES), N = 8192, interleaved bursts (scripts/gemm_ab.py)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for st in 4 5 6 7; do
  rm -f paper_2103_14409_b200/_build/gemm.cu.o
  LSCAT_NVCC_EXTRA="-DGEMM2_STAGES=$st" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null || { echo "build failed $st"; continue; }
  echo "stages $st $(timeout 120 python scripts/gemm_ab.py 192,256,512)"
done
rm -f paper_2103_14409_b200/_build/gemm.cu.o
