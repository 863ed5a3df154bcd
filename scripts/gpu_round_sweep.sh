cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_round.sh
timeout 900 python scripts/sweep_c4.py --out gpurun_out/r02_sweep_c4.json > gpurun_out/sweep.log 2>&1
