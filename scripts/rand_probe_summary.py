"""profiles/rand_probe.json from the ncu CSV of scripts/rand_probe (2^24
random reads per launch of width 4, 16, 32 B over a 1 GiB array): the random
read ceiling of this B200 and the DRAM bytes one random read costs.

    python scripts/rand_probe_summary.py gpurun_out/rand.csv profiles/rand_probe.json
"""
import csv
import json
import sys

N = 1 << 24
rows = {}
with open(sys.argv[1]) as f:
    for r in csv.DictReader(l for l in f if l.startswith('"')):
        rows.setdefault((r["ID"], r["Kernel Name"]), {})[r["Metric Name"]] = float(
            r["Metric Value"].replace(",", ""))
out = {"launch": "2^24 threads, one random W-aligned read each, 1 GiB array (scripts/rand_probe.cu)",
       "per_width": []}
for (i, name), m in sorted(rows.items()):
    t = m["gpu__time_duration.sum"] * 1e-9
    out["per_width"].append({"kernel": name, "time_us": t * 1e6,
                             "dram_bytes_per_read": m["dram__bytes_read.sum"] / N,
                             "reads_per_s": N / t})
best = max(out["per_width"], key=lambda w: w["reads_per_s"])
out["random_reads_per_s"] = best["reads_per_s"]
out["bytes_per_random_read"] = sum(w["dram_bytes_per_read"] for w in out["per_width"]) / len(out["per_width"])
with open(sys.argv[2], "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
