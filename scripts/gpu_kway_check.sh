#!/bin/bash
# one-pass cascade A/B: parity with it on, then the launch list of 64 C3 updates
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export GPULSM_KWAY_MIN_B=${KWAY:-32768}
timeout 1200 python -m pytest tests -m gpu -q ${PYX--x} --timeout 600 -k "not launch_counter ${PYTEST_K:+and $PYTEST_K}" > gpurun_out/pytest_kway.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_kway.log
P="python scripts/prof_step.py --no-cleanup --nq 1024"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/km_launches.csv $P > gpurun_out/km_list.log 2>&1
if [ -n "$FULL" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kmerge -s ${KS:-31} -c 1 -o gpurun_out/prof_km6 $P > gpurun_out/km_full.log 2>&1
fi
