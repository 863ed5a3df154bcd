"""Per-kernel totals and per-launch times from an ncu launch list CSV.

    python scripts/launch_table.py gpurun_out/km_launches.csv [kernel_regex]
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
T = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "").split("::")[-1]})
    v = float(r[vi].replace(",", ""))
    d[r[mi]] = v * T.get(r[ui], 1.0) if "time" in r[mi] else v
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in per.values():
    a = agg[d["name"]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} n={a[0]:5d} total {a[1]:10.1f} us ({100 * a[1] / tot:5.1f}%)  mean {a[1] / a[0]:8.2f} us  "
          f"DRAM {a[2] / max(a[1], 1e-9) / 1e3:7.1f} GB/s")
if len(sys.argv) > 2:
    pat = re.compile(sys.argv[2])
    print([round(d.get("gpu__time_duration.sum", 0), 1) for d in per.values() if pat.search(d["name"])])
