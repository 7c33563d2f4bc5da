cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tpb scripts/tp_band_probe.cu && { timeout 300 /tmp/tpb 8192; timeout 300 /tmp/tpb 4096; } > gpurun_out/tp_band.txt 2>&1
echo done
