#!/bin/bash
# Round-2 captures (run under gpurun from the repo root): racecheck minimal reproducer, ncu --set
# full of the CTA-pair GEMM, the cold euclid launch and the transpose at N = 8192, and the launch
# list of the bench command (tiny policy).
set -x
O=gpurun_out/r2
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/rc scripts/racecheck_tmem_pair.cu
compute-sanitizer --tool racecheck /tmp/rc 2 > $O/racecheck_min_pair.txt 2>&1
compute-sanitizer --tool racecheck /tmp/rc 1 > $O/racecheck_min_single.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:gemm_2cta -s 2 -c 1 -o $O/prof_gemm2cta -f python scripts/prof_launch.py gemm_bf16 8192 256 3 > $O/ncu_gemm.log 2>&1
$NCU -k regex:row_kernel -s 2 -c 1 -o $O/prof_euclid_cold -f python scripts/prof_launch.py euclid 8192 896 3 > $O/ncu_euclid.log 2>&1
$NCU -k regex:transpose -s 2 -c 1 -o $O/prof_transpose -f python scripts/prof_launch.py transpose 8192 256 3 > $O/ncu_transpose.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_tiny.csv \
  python bench.py --policy tiny --steps 1 --warmup 1 --no-secondary --no-e2e --no-cpu > $O/bench_tiny_under_ncu.log 2>&1
cuobjdump -sass paper_2103_14409_b200/liblscat.so > /tmp/sass.txt 2>/dev/null
for m in UTCHMMA "UTCHMMA.2CTA" UTMALDG UTMASTG LDTM STTM UBLKCP; do
  echo "$m $(grep -c "$m" /tmp/sass.txt)"; done > $O/sass_counts.txt
echo "HMMA(legacy) $(grep -cE '[^C]HMMA' /tmp/sass.txt)" >> $O/sass_counts.txt
echo done
