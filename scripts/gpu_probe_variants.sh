cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/probe_var.txt
for f in scripts/sp_*; do echo "=== $f" >> gpurun_out/probe_var.txt; timeout 60 $f >> gpurun_out/probe_var.txt 2>&1; done
