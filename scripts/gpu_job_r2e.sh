# round 2: fused / early percentile selection (R-27) — the new reduce tests + table timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_reduce.py -x -q -k "early or fused" > gpurun_out/pytest_reduce.log 2>&1; echo "reduce tests rc=$?"; tail -3 gpurun_out/pytest_reduce.log
timeout 600 python scripts/table_bench_early.py > gpurun_out/table_early.json 2> gpurun_out/table_early.err; echo "table rc=$?"
echo done
