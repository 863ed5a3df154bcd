#!/bin/bash
# full GPU tests + smoke + a short bench without the secondary configs (A/B turnaround)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_q.log
timeout 300 python scripts/overlap_handles.py > gpurun_out/overlap.log 2>&1
