#!/bin/bash
# C5 on one GPU (b = 2^24, 2^30 resident) + launch list of the multi-wave LSD sort
# and --set full captures of its passes at b = 2^21 and 2^24
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1
echo "c5 exit $?" >> gpurun_out/bench_c5.log
for B in 2097152 16777216; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lsd_launches_$B.csv python scripts/prof_step.py --b $B --batches 4 --nq 1024 --no-cleanup > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:onesweep_pass -s 4 -c 2 -o gpurun_out/prof_lsd_$B python scripts/prof_step.py --b $B --batches 4 --nq 1024 --no-cleanup > /dev/null 2>&1
done
