#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
{
for f in 0.35 0.4 0.45 0.5 0.55; do LSCAT_ROW_L2FRAC=$f timeout 300 python scripts/sweep_probe.py euclid 8192; done
rm -f paper_2103_14409_b200/_build/kern_rows.cu.o
LSCAT_NVCC_EXTRA="-DL2_SECONDARY_UNCHANGED" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null
echo '{"variant": "secondary evict_unchanged"}'
for f in 0.3 0.45 0.6 0.8; do LSCAT_ROW_L2FRAC=$f timeout 300 python scripts/sweep_probe.py euclid 8192; done
} > gpurun_out/l2frac2.jsonl 2>&1
rm -f paper_2103_14409_b200/_build/kern_rows.cu.o
echo done
