#!/bin/bash
# C4 long-range work: parity of the multi-level range/count paths, then the quick C4 sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -k "${PYTEST_K:-long_ranges or nine_levels or c4_shape or golden or edge_queries}" > gpurun_out/pytest_c4.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_c4.log
timeout 900 python scripts/sweep_c4.py ${SWEEP_ARGS:---quick} --out gpurun_out/sweep_c4.json > gpurun_out/sweep_c4.log 2>&1
echo "sweep exit $?" >> gpurun_out/sweep_c4.log
