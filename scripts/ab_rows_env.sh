#!/bin/bash
# A/B of the row-kernel grid (round-1 grid vs balanced), interleaved, same box session.
for i in 1 2; do
  LSCAT_ROW_GRID=legacy python scripts/ab_rows.py paper_2103_14409_b200/liblscat.so legacy_grid
  python scripts/ab_rows.py paper_2103_14409_b200/liblscat.so balanced_grid
done
