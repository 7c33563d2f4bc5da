#!/bin/bash
# One GPU session: build, tests, smoke, bench, optional ncu captures.  Usage:
#   scripts/gpu_round.sh [tests] [smoke] [bench_fast] [bench] [ncu_reduce] [ncu_euclid] [ncu_gemm] [launches] [suite]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
for job in "$@"; do
  case $job in
    tests) timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_gpu.log ;;
    smoke) timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log ;;
    bench_fast) timeout 600 python bench.py --policy fast > gpurun_out/bench_fast.log 2>&1; echo "bench_fast rc=$?" ;;
    bench) timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" ;;
    ncu_reduce) timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_ -c 1 -o gpurun_out/prof_reduce -f python scripts/profile_kernels.py reduce 100000000 > gpurun_out/ncu_reduce.log 2>&1; echo "ncu_reduce rc=$?" ;;
    ncu_euclid) timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_kernel -c 2 -o gpurun_out/prof_euclid -f python scripts/profile_kernels.py euclid8192 512 > gpurun_out/ncu_euclid.log 2>&1; echo "ncu_euclid rc=$?" ;;
    ncu_euclid32) timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_kernel -c 2 -o gpurun_out/prof_euclid32 -f python scripts/profile_kernels.py euclid8192 32 > gpurun_out/ncu_euclid32.log 2>&1; echo "ncu_euclid32 rc=$?" ;;
    ncu_steady) timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:row_kernel --csv --log-file gpurun_out/euclid_steady.csv python scripts/profile_kernels.py euclid8192 32 30 > gpurun_out/ncu_steady.log 2>&1; echo "ncu_steady rc=$?" ;;
    ncu_euclid_steady_full) timeout 1500 ncu --set full --replay-mode application --cache-control none --clock-control none --import-source on -k regex:row_kernel -s 20 -c 1 -o gpurun_out/prof_euclid32_steady -f python scripts/profile_kernels.py euclid8192 32 24 > gpurun_out/ncu_euclid_steady_full.log 2>&1; echo "ncu_euclid_steady_full rc=$?" ;;
    ncu_transpose) timeout 600 ncu --set full --clock-control none --import-source on -k regex:transpose -c 1 -s 1 -o gpurun_out/prof_transpose -f python scripts/profile_kernels.py kernel transpose 8192 512 > gpurun_out/ncu_tp.log 2>&1; echo "ncu_transpose rc=$?" ;;
    ncu_gemm) timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/prof_gemm -f python scripts/profile_kernels.py gemm8192 256 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu_gemm rc=$?" ;;
    launches) timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --policy tiny --steps 1 --warmup 0 --no-e2e --no-secondary --no-cpu > gpurun_out/launches_bench.log 2>&1; echo "launches rc=$?" ;;
    ncu_select) timeout 900 ncu --set full --clock-control none --import-source on -k regex:sel_pass -c 3 -o gpurun_out/prof_select -f python scripts/profile_kernels.py reduce 1000000000 > gpurun_out/ncu_select.log 2>&1; echo "ncu_select rc=$?" ;;
    stats_list) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/stats_list.csv python scripts/profile_kernels.py reduce 1000000000 > gpurun_out/ncu_stats.log 2>&1; echo "stats_list rc=$?" ;;
    suite) timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/suite8192.csv python scripts/profile_kernels.py suite8192 > gpurun_out/ncu_suite.log 2>&1; echo "suite rc=$?" ;;
  esac
done
