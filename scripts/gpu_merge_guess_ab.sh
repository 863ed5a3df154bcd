cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "golden or c1 or schedule or ragged or multi_tile or concentrated or cascade or nine or sa or bulk or update_batches" > gpurun_out/pytest_mg.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_mg.log
for G in 1 0; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DGPULSM_PROBE -DMERGE_GUESS=1 -DMERGE_GUESS_TILE=$G -I include -I paper_1707_05354_b200/csrc scripts/merge_probe.cu -o /tmp/mp$G > /dev/null 2>&1
  echo "== MERGE_GUESS_TILE=$G" >> gpurun_out/mprobe.txt
  (/tmp/mp$G 2097152; /tmp/mp$G 8388608; /tmp/mp$G 33554432) 2>&1 | grep -E "merge avg|search0|search1|c_search|done" >> gpurun_out/mprobe.txt
done
VARIANTS="libgpulsm.so libgpulsm_notile.so" bash scripts/gpu_ab_variants.sh
