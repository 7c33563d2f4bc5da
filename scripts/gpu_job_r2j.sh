cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
LSCAT_SEL_DEBUG=1 timeout 300 python scripts/early_probe.py 1000000000 3 > gpurun_out/early_probe.txt 2>&1; echo "probe rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/early_1e9_launches.csv python scripts/early_probe.py 1000000000 2 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 python scripts/table_bench_early.py > gpurun_out/table_early.json 2> gpurun_out/table_early.err; echo "table rc=$?"
timeout 1800 python -m pytest tests/test_gpu_reduce.py -x -q -k "sampled or early or percentiles or scaled" > gpurun_out/pytest_reduce.log 2>&1; echo "reduce tests rc=$?"; tail -3 gpurun_out/pytest_reduce.log
echo done
