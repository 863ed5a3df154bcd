"""Per-CUDA-line instruction and stall-sample totals from an ncu report
(needs -lineinfo and --import-source on):

    python scripts/ncu_lines.py REP KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                               "--kernel-name", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                              text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
fname, res, hdr = None, [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name" or r[2] != "-":
        continue  # keep CUDA-line rows (Address == "-")
    try:
        ins = float(r[hdr.index("Instructions Executed")])
        smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    res.append((fname, r[0], r[1].strip()[:70], ins, smp))
ti = sum(x[3] for x in res) or 1
ts = sum(x[4] for x in res) or 1
print(f"total instructions {ti:.3e}  samples {ts:.0f}")
for f, ln, src, ins, smp in sorted(res, key=lambda x: -x[4])[:top]:
    print(f"{f}:{ln:>4} inst {100 * ins / ti:5.1f}% stall {100 * smp / ts:5.1f}%  {src}")
