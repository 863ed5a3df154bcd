# A/B of two in-tree library builds (one GPU call): gpu tests on the default
# build, the bench with each, and ncu DRAM bytes of the query kernels with each.
# Usage: AB_LIB=libgpulsm_<name>.so bash scripts/gpu_ab_lib.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 800 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_a.log 2>&1
timeout 800 env GPULSM_LIB=$AB_LIB python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_b.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
K='regex:lookup_kernel|count_kernel|range_block'
timeout 600 ncu --metrics $M --clock-control none -k "$K" --csv --log-file gpurun_out/q_a.csv python scripts/prof_step.py > /dev/null 2>&1
timeout 600 env GPULSM_LIB=$AB_LIB ncu --metrics $M --clock-control none -k "$K" --csv --log-file gpurun_out/q_b.csv python scripts/prof_step.py > /dev/null 2>&1
