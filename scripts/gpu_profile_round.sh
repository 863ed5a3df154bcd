# Round profile: full bench line, ncu launch list of the bench command, and
# --set full captures of the top kernels (one GPU; no multi-rank commands).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/clocks_before.csv 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/ncu_list.log 2>&1
P="python scripts/prof_step.py"
NCU="timeout 600 ncu --set full --clock-control none --import-source on"
$NCU -k regex:^count_kernel -s 0 -c 2 -o gpurun_out/prof_count $P > /dev/null 2>&1
$NCU -k regex:range_block -s 0 -c 2 -o gpurun_out/prof_range $P > /dev/null 2>&1
$NCU -k regex:lookup -s 0 -c 2 -o gpurun_out/prof_lookup $P > /dev/null 2>&1
$NCU -k regex:merge_kernel -s 62 -c 1 -o gpurun_out/prof_merge $P --no-cleanup --nq 1024 > /dev/null 2>&1
$NCU -k regex:merge_kernel -s 0 -c 1 -o gpurun_out/prof_merge0 $P --batches 4 --no-cleanup --nq 1024 > /dev/null 2>&1
$NCU -k regex:msd_scatter -s 60 -c 1 -o gpurun_out/prof_sort $P --no-cleanup --nq 1024 > /dev/null 2>&1
$NCU -k regex:bucket_rank -s 60 -c 1 -o gpurun_out/prof_bucket $P --no-cleanup --nq 1024 > /dev/null 2>&1
$NCU -k regex:cleanup_write -s 0 -c 1 -o gpurun_out/prof_cleanup $P --nq 1024 > /dev/null 2>&1
# summarise on the box (the reports are too big to bring back): profiles
# summaries under gpurun_out/prof_summary, reports deleted except small ones
python scripts/ncu_summary.py --launches gpurun_out/launches.csv --reps "gpurun_out/prof_*.ncu-rep" \
    --round ${ROUND:-r01} --outdir gpurun_out/prof_summary > gpurun_out/ncu_summary.log 2>&1
mkdir -p gpurun_out/keep
for f in prof_range prof_bucket prof_merge; do mv gpurun_out/$f.ncu-rep gpurun_out/keep/ 2>/dev/null; done
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out/* | sort -h | tail -20
# sort timeline probe and the C4 query sweep
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DGPULSM_PROBE -I include -I paper_1707_05354_b200/csrc scripts/msd_probe.cu -o /tmp/msd_probe > /dev/null 2>&1
timeout 120 /tmp/msd_probe > gpurun_out/msd_probe.txt 2>&1
timeout 900 python scripts/sweep_c4.py --out gpurun_out/${ROUND:-r01}_sweep_c4.json > gpurun_out/sweep.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/rand_probe.cu -o /tmp/rand_probe > /dev/null 2>&1
timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/rand.csv /tmp/rand_probe > /dev/null 2>&1
python scripts/rand_probe_summary.py gpurun_out/rand.csv gpurun_out/rand_probe.json > /dev/null 2>&1
