#!/bin/bash
# A/B of several in-tree library builds: the C3 bench (update phase) with each,
# interleaved twice. Usage: AB_LIBS="libgpulsm.so libgpulsm_x.so ..." bash scripts/gpu_ab_multi.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/ab_multi.log
for rep in 1 2; do
  for L in $AB_LIBS; do
    timeout 600 env GPULSM_LIB=$L python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/ab_one.log 2>&1
    python - "$L" >> gpurun_out/ab_multi.log <<'PY'
import json, sys
l = [x for x in open("gpurun_out/ab_one.log") if x.startswith("{")]
if l:
    d = json.loads(l[-1])
    print(sys.argv[1], round(d["value"], 1), round(d["phase_ms"]["update"], 4), round(d["ms_per_step"], 3))
else:
    print(sys.argv[1], "FAILED", open("gpurun_out/ab_one.log").read()[-300:].replace("\n", " "))
PY
  done
done
