#!/bin/bash
# the driver's round-end order on one box: GPU tests, smoke, then the bench
# (twice here: does the first bench after the tests run slower?)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
for i in 1 2; do
  nvidia-smi --query-gpu=temperature.gpu,temperature.memory,power.draw,clocks.sm,clocks.mem,clocks_event_reasons.active --format=csv > gpurun_out/nvsmi_$i.csv 2>&1
  timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_fresh$i.log 2>&1
done
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
echo "c5 exit $?" >> gpurun_out/bench_c5.log
