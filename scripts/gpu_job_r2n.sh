# sel_small grid calibration: keys per CTA (LSCAT_SMALL_KEYS_PER_CTA), small tables only
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_reduce.py -x -q -k "not 1e9 and not sampled" > gpurun_out/pytest_reduce.log 2>&1; echo "reduce tests rc=$?"; tail -2 gpurun_out/pytest_reduce.log
for v in 512 2048 4096 8192 16384; do
  echo "keys_per_cta=$v"
  LSCAT_SMALL_KEYS_PER_CTA=$v LSCAT_TABLE_SMALL_ONLY=1 timeout 300 python scripts/table_bench_early.py 2>&1 >/dev/null | grep -v "^$"
done > gpurun_out/small_grid.txt 2>&1
echo done
