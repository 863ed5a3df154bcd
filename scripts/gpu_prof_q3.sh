# ncu --set full of the 3-level (post-cleanup) range and count launches of a
# C3 cycle, with source-level stall data (one GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU="timeout 900 ncu --set full --clock-control none --import-source on"
$NCU -k regex:range_block -s 1 -c 1 -o gpurun_out/prof_range3 python scripts/prof_step.py > /dev/null 2>&1
$NCU -k regex:count_kernel -s 1 -c 1 -o gpurun_out/prof_count3 python scripts/prof_step.py > /dev/null 2>&1
for r in range3 count3; do
  python scripts/ncu_sass_top.py gpurun_out/prof_$r.ncu-rep 40 > gpurun_out/prof_${r}_sass.txt 2>&1
  python scripts/ncu_lines.py gpurun_out/prof_$r.ncu-rep '.*' 0 40 > gpurun_out/prof_${r}_lines.txt 2>&1
done
