#!/bin/bash
# sort timeline probe (%globaltimer stamps per phase)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DGPULSM_PROBE -I include -I paper_1707_05354_b200/csrc scripts/msd_probe.cu -o /tmp/msd_probe > gpurun_out/probe_build.log 2>&1
timeout 120 /tmp/msd_probe ${PROBE_B:-1048576} > gpurun_out/msd_probe.txt 2>&1
