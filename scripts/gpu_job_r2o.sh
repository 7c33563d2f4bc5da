cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_reduce.log 2>&1; echo "reduce tests rc=$?"; tail -2 gpurun_out/pytest_reduce.log
timeout 600 python scripts/table_bench_early.py > gpurun_out/table_early.json 2> gpurun_out/table_early.err; echo "table rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/early_1e9_launches.csv python scripts/early_probe.py 1000000000 2 > /dev/null 2>&1; echo "ncu rc=$?"
echo done
