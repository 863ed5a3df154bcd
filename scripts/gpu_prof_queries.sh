# ncu --set full captures of the query kernels (before and after cleanup)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="python scripts/prof_step.py"
NCU="timeout 900 ncu --set full --clock-control none --import-source on"
$NCU -k regex:^range_kernel -s 0 -c 2 -o gpurun_out/prof_range $P > gpurun_out/ncu_q.log 2>&1
$NCU -k regex:^count_kernel -s 0 -c 2 -o gpurun_out/prof_count $P >> gpurun_out/ncu_q.log 2>&1
$NCU -k regex:^lookup_kernel -s 0 -c 2 -o gpurun_out/prof_lookup $P >> gpurun_out/ncu_q.log 2>&1
