cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "long_ranges_multi or nine or schedule or c1 or golden" > gpurun_out/pytest_lk.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_lk.log
for L in libgpulsm.so libgpulsm_ln4.so; do echo "== $L"; GPULSM_LIB=$L timeout 600 python scripts/lookup_levels.py; done > gpurun_out/lookup_levels.log 2>&1

