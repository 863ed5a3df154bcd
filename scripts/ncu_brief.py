"""Key counters + stall samples + top source lines of one ncu report.

    python scripts/ncu_brief.py REP KERNEL_REGEX [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                              stderr=subprocess.DEVNULL)
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
keys = ("gpu__time_duration.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size")
for k, x in zip(h, v):
    if k in keys:
        print(f"{k:60s} {x} {r[1][h.index(k)]}")
st = [(k, float(x.replace(",", ""))) for k, x in zip(h, v)
      if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
tot = sum(x for _, x in st) or 1
for k, x in sorted(st, key=lambda t: -t[1])[:8]:
    print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * x / tot:5.1f}%")
subprocess.call([sys.executable, __file__.replace("ncu_brief.py", "ncu_lines.py"), rep, kern, "0", str(top)])
