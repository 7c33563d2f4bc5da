#!/bin/bash
# row kernels: persistent grid for B > 512 (ROW_PERSIST_BIG=1) vs one pass (0); PDL sweep probe
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sweep.py -q -x -k "vector or euclid or pdl or bench_launch" 2>&1 | tail -1
{
timeout 300 python scripts/sweep_probe.py euclid 4096,8192
rm -f paper_2103_14409_b200/_build/kern_rows.cu.o
LSCAT_NVCC_EXTRA="-DROW_PERSIST_BIG=0" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null
echo '{"variant": "ROW_PERSIST_BIG=0"}'
timeout 300 python scripts/sweep_probe.py euclid 4096,8192
} > gpurun_out/row_persist.jsonl 2>&1
rm -f paper_2103_14409_b200/_build/kern_rows.cu.o
echo done
