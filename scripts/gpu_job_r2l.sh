cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python scripts/table_bench_early.py > gpurun_out/table_early.json 2> gpurun_out/table_early.err; echo "table rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/small_launches.csv python scripts/small_table_probe.py 2140796 3 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_gpu.log
echo done
