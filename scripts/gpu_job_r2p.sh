# row kernels at N = 4096: the 4-deep variant (occupancy-sized grid) against the 8-deep one, interleaved
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
for i in 1 2; do
  AB_BY_BLOCK=1 LSCAT_ROW_SMALL4_MAX=2048 python scripts/ab_rows.py paper_2103_14409_b200/liblscat.so deep8_at_4096
  AB_BY_BLOCK=1 LSCAT_ROW_SMALL4_MAX=4096 python scripts/ab_rows.py paper_2103_14409_b200/liblscat.so deep4_at_4096
done > gpurun_out/ab_4096.jsonl 2>&1
echo done
