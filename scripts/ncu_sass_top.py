"""Top SASS instructions of an ncu report by stall samples, with the CUDA
line and the main stall reasons.   python scripts/ncu_sass_top.py REP [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                               "sass"], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
hdr, start = None, 0
for i, r in enumerate(rows[:5]):
    if r and r[0] == "Address":
        hdr, start = r, i + 1
res, tot = [], 0.0
for r in rows[start:]:
    d = dict(zip(hdr, r))
    try:
        smp = float(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    tot += smp
    st = {k[6:]: float(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v not in ("0", "")}
    res.append((smp, d["Address"], d["Source"].strip()[:48], sorted(st.items(), key=lambda x: -x[1])[:2]))
res.sort(key=lambda x: -x[0])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for smp, a, src, st in res[:n]:
    print(f"{100 * smp / tot:5.1f}% {a} {src:48s} {st}")
