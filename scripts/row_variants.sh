#!/bin/bash
# Row-kernel register-budget / loads-in-flight variants: rebuild kern_rows.cu with each
# (-D) setting and time euclid at every block size (scripts/row_probe_all.py), N = 8192 and 4096.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "ROW_MINB_THREADS=2048" "ROW_MINB_THREADS=1024" "ROW_MINB_THREADS=768" "ROW_MINB_THREADS=640" "ROW_MINB_THREADS=1024 -DROW_U=4" "ROW_MINB_THREADS=768 -DROW_U=6"; do
  rm -f paper_2103_14409_b200/_build/kern_rows.cu.o
  LSCAT_NVCC_EXTRA="-D$v" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null || { echo "build failed $v"; continue; }
  for tw in auto 1 2; do
    for n in 8192 4096; do
      if [ $tw = auto ]; then r=$(N=$n timeout 120 python scripts/row_probe_all.py); else r=$(LSCAT_ROW_TEAM_WARPS=$tw N=$n timeout 120 python scripts/row_probe_all.py); fi
      echo "{\"variant\": \"$v\", \"tw\": \"$tw\", \"res\": $r}"
    done
  done
done | tee gpurun_out/row_variants.jsonl
rm -f paper_2103_14409_b200/_build/kern_rows.cu.o
