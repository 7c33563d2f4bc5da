#!/bin/bash
# calibration grid for the row kernels (euclid): warps/SM cap x team warps
cd "$(dirname "$0")/.."
for cap in 0 16 24 32 48; do
  for tw in auto 1 2 4; do
    if [ $tw = auto ]; then LSCAT_ROW_WARPS_PER_SM=$cap python scripts/row_tw_probe.py | sed "s/^/cap=$cap /";
    else LSCAT_ROW_WARPS_PER_SM=$cap LSCAT_ROW_TEAM_WARPS=$tw python scripts/row_tw_probe.py | sed "s/^/cap=$cap /"; fi
  done
done
for n in 4096 2048; do N=$n python scripts/row_tw_probe.py | sed "s/^/default /"; done
