#!/bin/bash
# CTA-pair GEMM rasterisation group height (GEMM2_GROUPM), N = 8192 (calibration)
cd "$(dirname "$0")/.."
for gm in 4 8 16 32; do
  rm -f paper_2103_14409_b200/_build/gemm.cu.o
  LSCAT_NVCC_EXTRA="-DGEMM2_GROUPM=$gm" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null || { echo "build failed $gm"; continue; }
  echo "groupm $gm $(timeout 120 python scripts/gemm_ab.py 192,256)"
done
rm -f paper_2103_14409_b200/_build/gemm.cu.o
