cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# launch list (all kernels, device time, cold & serialised)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python scripts/prof_step.py > gpurun_out/ncu_list.log 2>&1
echo "list exit $?" >> gpurun_out/ncu_list.log
# full captures: merges of the 64th insert (skip 57), one onesweep pass, hist, lookup, count
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_kernel -s 57 -c 6 -o gpurun_out/merge_r01 python scripts/prof_step.py --no-cleanup > gpurun_out/ncu_merge.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep -s 200 -c 2 -o gpurun_out/sort_r01 python scripts/prof_step.py --no-cleanup > gpurun_out/ncu_sort.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sort_hist|lookup_kernel|count_kernel" -s 50 -c 3 -o gpurun_out/misc_r01 python scripts/prof_step.py --no-cleanup > gpurun_out/ncu_misc.log 2>&1
ls -la gpurun_out
