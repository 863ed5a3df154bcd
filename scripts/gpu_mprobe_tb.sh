cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(./scripts/merge_probe 1048576; ./scripts/merge_probe 4194304; ./scripts/merge_probe 33554432) > gpurun_out/mprobe.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
