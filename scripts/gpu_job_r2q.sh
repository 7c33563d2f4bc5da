cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sel_pass_sampled" -c 1 -o gpurun_out/prof_pass -f python scripts/early_probe.py 1000000000 1 > gpurun_out/ncu_pass.log 2>&1; echo "ncu rc=$?"
echo done
