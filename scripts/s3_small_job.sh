#!/bin/bash
# Session-3 small-table probe: phase stamps of sel_small (LSCAT_SEL_DEBUG), event timing of
# reduce + 9 percentiles (early path), optional ncu launch list / --set full captures.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for w in gtx980 t4; do
  LSCAT_SEL_DEBUG=1 timeout 300 python scripts/small_early_probe.py $w 4 > $O/dbg_$w.log 2>&1
  timeout 300 python scripts/small_early_probe.py $w 12 > $O/time_$w.log 2>&1
  if [ "$1" = ncu ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv python scripts/small_early_probe.py $w 4 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reduce_groups|sel_small" -s 6 -c 2 -o $O/prof_small_$w -f python scripts/small_early_probe.py $w 6 > $O/ncu_$w.log 2>&1
  fi
done
grep -h "phases\|total" $O/dbg_*.log $O/time_*.log | tail -40
