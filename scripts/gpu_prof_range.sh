cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="python scripts/prof_step.py --no-cleanup"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"range_write|count_kernel" -s 1 -c 2 -o gpurun_out/prof_rw $P > gpurun_out/ncu_rw.log 2>&1
