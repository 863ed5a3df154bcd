cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"count_kernel|range_block" -c 2 -o gpurun_out/c4_l1024 python scripts/prof_c4.py --r 127 --L 1024 > gpurun_out/c4prof.log 2>&1
echo "exit $?" >> gpurun_out/c4prof.log
