cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tpb scripts/tp_band_probe.cu && { /tmp/tpb 8192; /tmp/tpb 4096; } > gpurun_out/tp_band.txt 2>&1
timeout 300 python scripts/small_table_probe.py 2140796 8 > gpurun_out/small_probe.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_launches.csv python scripts/small_table_probe.py 2140796 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small5m_launches.csv python scripts/small_table_probe.py 5028536 3 > /dev/null 2>&1
echo done
