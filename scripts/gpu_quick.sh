#!/bin/bash
# quick A/B: GPU parity subset + the launch list of 64 C3 updates (+ optional bench)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q ${PYX--x} --timeout 600 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_q.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_q.log
P="python scripts/prof_step.py --no-cleanup --nq 1024"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv $P > gpurun_out/q_list.log 2>&1
if [ -n "$BENCH" ]; then timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; fi
if [ -n "$FULLK" ]; then timeout 600 ncu --set full --clock-control none --cache-control ${CACHE:-all} --import-source on -k regex:$FULLK -s ${KS:-60} -c 1 -o gpurun_out/prof_q $P > gpurun_out/q_full.log 2>&1; fi
