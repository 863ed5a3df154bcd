cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/rank.txt
for v in 0 1 2; do echo "=== variant $v" >> gpurun_out/rank.txt; timeout 60 ./scripts/sp_rank$v >> gpurun_out/rank.txt 2>&1; done
