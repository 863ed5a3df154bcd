cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(timeout 60 ./scripts/sort_probe; LSD_ONLY=1 timeout 60 ./scripts/sort_probe; timeout 60 ./scripts/sort_probe 5000) 2>&1 | grep -E "sort avg|err=" > gpurun_out/probe.txt
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
