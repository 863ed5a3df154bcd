# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_run.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SAN_BIG=1 timeout 1500 $CS --tool memcheck --leak-check no python scripts/sanitize_run.py > gpurun_out/sanitizer_memcheck.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer_memcheck.log
timeout 1500 $CS --tool racecheck python scripts/sanitize_run.py > gpurun_out/sanitizer_racecheck.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer_racecheck.log
SAN_BIG=1 timeout 1500 $CS --tool synccheck python scripts/sanitize_run.py > gpurun_out/sanitizer_synccheck.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer_synccheck.log
