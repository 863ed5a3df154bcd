#!/bin/bash
# merge-kernel A/B: merge-related parity tests, the merge probe built from the
# current sources, and the bench with $VARIANTS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "golden or c1 or schedule or ragged or multi_tile or concentrated or cascade or nine or sa or bulk or update_batches or tiny" > gpurun_out/pytest_mg.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_mg.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DGPULSM_PROBE -I include -I paper_1707_05354_b200/csrc scripts/merge_probe.cu -o /tmp/mp > /dev/null 2>&1
(/tmp/mp 1048576; /tmp/mp 2097152; /tmp/mp 8388608; /tmp/mp 33554432) 2>&1 | grep -E "merge avg|c_search" > gpurun_out/mprobe.txt
bash scripts/gpu_ab_variants.sh
