# sort kernels: ncu --set full of one msd_scatter and one bucket_rank launch
# (batch 6 of a C3 run), the random-read probe, and an A/B bench of a variant
# library (AB_LIB). One GPU.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/rand.csv scripts/rand_probe > /dev/null 2>&1
python scripts/rand_probe_summary.py gpurun_out/rand.csv gpurun_out/rand_probe.json > /dev/null 2>&1
NCU="timeout 600 ncu --set full --clock-control none --import-source on"
$NCU -k regex:msd_scatter -s 6 -c 1 -o gpurun_out/prof_msd python scripts/prof_step.py --batches 8 --nq 1024 --no-cleanup > /dev/null 2>&1
$NCU -k regex:bucket_rank -s 6 -c 1 -o gpurun_out/prof_brank python scripts/prof_step.py --batches 8 --nq 1024 --no-cleanup > /dev/null 2>&1
for r in msd brank; do
  ncu -i gpurun_out/prof_$r.ncu-rep --page details --csv > gpurun_out/prof_${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_$r.ncu-rep --page source --csv > gpurun_out/prof_${r}_source.csv 2>/dev/null
done
if [ -n "$AB_LIB" ]; then
  timeout 800 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_a.log 2>&1
  timeout 800 env GPULSM_LIB=$AB_LIB python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_b.log 2>&1
fi
