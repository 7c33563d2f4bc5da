cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_reduce.py -x -q -k "sampled or early or percentiles" > gpurun_out/pytest_reduce.log 2>&1; echo "reduce tests rc=$?"; tail -3 gpurun_out/pytest_reduce.log
for v in 1 3 4; do
  rm -f paper_2103_14409_b200/_build/stats.cu.o
  LSCAT_NVCC_EXTRA="-DSP_MINB=$v" python -c "import paper_2103_14409_b200.build as b; b.build()" > /dev/null 2>&1
  echo "SP_MINB=$v"
  LSCAT_SEL_DEBUG=1 timeout 300 python scripts/early_probe.py 1000000000 4 2>&1 | grep -E "rep |sel_finish"
  timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:sel_pass_sampled --csv python scripts/early_probe.py 1000000000 1 2>/dev/null | grep -E "sel_pass" | cut -c1-40,200-400
done > gpurun_out/spminb.txt 2>&1
echo done
