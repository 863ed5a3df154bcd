"""Summarise an ncu --metrics CSV: per kernel launch, duration and metrics."""
import csv
import sys
from collections import defaultdict

rows = defaultdict(dict)
order = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    key = (r["ID"], r["Kernel Name"][:40])
    if key not in rows:
        order.append(key)
    rows[key][r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
for key in order:
    m = rows[key]
    print(key[0], key[1], " ".join(f"{k.split('__')[1][:22]}={v[0]}{v[1]}" for k, v in sorted(m.items())))
