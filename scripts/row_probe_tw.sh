#!/bin/bash
cd "$(dirname "$0")/.."
for tw in auto 1 2 4 8; do
  if [ $tw = auto ]; then python scripts/row_tw_probe.py; else LSCAT_ROW_TEAM_WARPS=$tw python scripts/row_tw_probe.py; fi
done
for n in 4096 2048 1024; do N=$n python scripts/row_tw_probe.py; done
