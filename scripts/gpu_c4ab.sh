#!/bin/bash
# C4 A/B: parity of the long-range paths on the default build, then the quick
# C4 sweep with the default build and with $AB_LIB
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -k "${PYTEST_K:-long_ranges or nine_levels or c4_shape or golden or edge_queries or schedule or c1 or concentrated}" > gpurun_out/pytest_c4.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_c4.log
timeout 900 python scripts/sweep_c4.py ${SWEEP_ARGS:---quick} > gpurun_out/sweep_a.log 2>&1
timeout 900 env GPULSM_LIB=$AB_LIB python scripts/sweep_c4.py ${SWEEP_ARGS:---quick} > gpurun_out/sweep_b.log 2>&1
