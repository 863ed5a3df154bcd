#!/bin/bash
# A/B of library variants on one-level C4 rows (r = 128) and the C3 bench:
# VARIANTS="libgpulsm.so libgpulsm_x.so ..."
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "${PYTEST_K:-long_ranges or golden or edge_queries or c1 or ragged}" > gpurun_out/pytest_ab.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_ab.log
: > gpurun_out/capab.log
for L in $VARIANTS; do
  echo "== $L" >> gpurun_out/capab.log
  GPULSM_LIB=$L timeout 600 python scripts/sweep_c4.py --rs ${RS:-128} --ls ${LS:-8,16,32,64,128,1024} >> gpurun_out/capab.log 2>&1
  v=$(timeout 600 env GPULSM_LIB=$L python bench.py --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); q=d['queries']; print('bench', round(d['value'],1), round(d['ms_per_step'],3), [round(q[k]) for k in ('lookup_mqps_before_cleanup','count_mqps_before_cleanup','range_mqps_before_cleanup','count_mqps_after_cleanup','range_mqps_after_cleanup')])")
  echo "$v" >> gpurun_out/capab.log
done
