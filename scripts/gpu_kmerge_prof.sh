#!/bin/bash
# kmerge A/B: launch list (per-launch times) of 64 C3 updates with the one-pass
# cascade on, and a --set full capture of the t = 6 kmerge
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export GPULSM_KWAY_MIN_B=${KWAY:-1}
P="python scripts/prof_step.py --no-cleanup --nq 1024"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/km_launches.csv $P > gpurun_out/km_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kmerge -s 31 -c 1 -o gpurun_out/prof_km6 $P > gpurun_out/km_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kmerge -s 0 -c 1 -o gpurun_out/prof_km1 $P >> gpurun_out/km_full.log 2>&1
