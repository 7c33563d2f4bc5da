# sampled pass gap counters: per-thread shared words (SP_GAPS=1, default) vs packed registers (0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_reduce.py -x -q -k "sampled or early or scaled or percentiles" > gpurun_out/pytest_reduce.log 2>&1; echo "reduce tests rc=$?"; tail -2 gpurun_out/pytest_reduce.log
for v in 1 0 1 0; do
  rm -f paper_2103_14409_b200/_build/stats.cu.o
  LSCAT_NVCC_EXTRA="-DSP_GAPS=$v" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null 2>&1
  echo "SP_GAPS=$v"
  timeout 300 python scripts/early_probe.py 1000000000 4 2>&1 | grep -E "rep [23]"
  timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:sel_pass_sampled --csv python scripts/early_probe.py 1000000000 1 2>/dev/null | grep -E "sel_pass" | awk -F'","' '{print $(NF-2), $NF}'
done > gpurun_out/spgaps.txt 2>&1
echo done
