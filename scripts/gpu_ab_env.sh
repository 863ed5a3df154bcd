# A/B of env settings on the default build (one GPU call): ncu DRAM bytes of
# the query kernels and the bench, for each setting in AB_ENVS (space-separated
# NAME=VALUE, "-" = none). Usage: AB_ENVS="- GPULSM_L2FETCH=32" bash scripts/gpu_ab_env.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -n "$RUN_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
K=${NCU_K:-'regex:lookup_kernel|count_kernel|range_block'}
i=0
for E in $AB_ENVS; do
  [ "$E" = "-" ] && E="GPULSM_NONE=1"
  timeout 800 env $E python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$i.log 2>&1
  timeout 600 env $E ncu --metrics $M --clock-control none -k "$K" -c 12 --csv --log-file gpurun_out/q_$i.csv python scripts/prof_step.py > /dev/null 2>&1
  echo "$i $E" >> gpurun_out/ab_index.txt
  i=$((i+1))
done
