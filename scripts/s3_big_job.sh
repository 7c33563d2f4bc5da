#!/bin/bash
# Session-3 10^9-row probe: stage events of the sampled selection, a launch list, and ncu
# --set full of the selection's small kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3b
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
LSCAT_SEL_TIMING=1 LSCAT_SEL_DEBUG=1 timeout 300 python scripts/early_probe.py 1000000000 4 > $O/timing.log 2>&1
timeout 300 python scripts/early_probe.py 1000000000 6 > $O/plain.log 2>&1
if [ "$1" = ncu ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python scripts/early_probe.py 1000000000 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sel_plan|sel_check|sel_finish|sel_slot|sel_sample" -s 5 -c 5 -o $O/prof_sel -f python scripts/early_probe.py 1000000000 2 > $O/ncu.log 2>&1
fi
cat $O/plain.log; grep -v "^  " $O/timing.log | tail -30
