#!/bin/bash
# Session-3: reduce + kernel roll-up + 9 percentiles on configs[2]/[3]: timing, launch list,
# ncu --set full of the roll-up kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3r
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for w in gtx980 t4; do
  timeout 300 python scripts/small_early_probe.py $w 12 1 > $O/time_$w.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv python scripts/small_early_probe.py $w 4 1 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rollup" -s 4 -c 2 -o $O/prof_rollup_$w -f python scripts/small_early_probe.py $w 4 1 > $O/ncu_$w.log 2>&1
done
for f in $O/time_*.log; do tail -4 $f; done
