#!/bin/bash
# sort A/B: sort-related parity tests, the MSD probe built from the current
# sources, and the bench with $VARIANTS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "ragged or multi_tile or multi_wave or skew or duplicate or one_wave or two_level or c1 or golden or tiny or partial or lsd or bulk or update_batches" > gpurun_out/pytest_sort.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_sort.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DGPULSM_PROBE -I include -I paper_1707_05354_b200/csrc scripts/msd_probe.cu -o /tmp/msd_probe > /dev/null 2>&1
timeout 120 /tmp/msd_probe > gpurun_out/msd_probe.txt 2>&1
bash scripts/gpu_ab_variants.sh
