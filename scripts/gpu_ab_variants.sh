#!/bin/bash
# bench A/B of in-tree library variants: VARIANTS="libgpulsm.so libgpulsm_x.so ..." (two rounds)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/ab_variants.log
for rep in 1 2; do
  for L in $VARIANTS; do
    v=$(timeout 600 env GPULSM_LIB=$L python bench.py --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); q=d['queries']; print(round(d['value'],1), round(d['ms_per_step'],3), [int(q[k]) for k in ('lookup_mqps_before_cleanup','count_mqps_before_cleanup','range_mqps_before_cleanup','lookup_mqps_after_cleanup','count_mqps_after_cleanup','range_mqps_after_cleanup')], round(d['cleanup']['ms'],3))")
    echo "$rep $L $v" >> gpurun_out/ab_variants.log
  done
done
