"""Side-by-side of two sweep_c4.py logs: python scripts/sweep_cmp.py A.log B.log"""
import json
import sys


def rows(path):
    out = {}
    for line in open(path):
        if line.startswith("{"):
            d = json.loads(line)
            out[(d["r"], d["L"])] = d
    return out


a, b = rows(sys.argv[1]), rows(sys.argv[2])
print(f"{'r':>4} {'lv':>2} {'L':>5} | {'count A':>9} {'count B':>9} | {'range A':>9} {'range B':>9}  (M q/s)")
for k in sorted(a):
    x, y = a[k], b.get(k)
    if y is None:
        continue
    print(f"{k[0]:4d} {x['levels']:2d} {k[1]:5d} | {x['count_mqps']:9.1f} {y['count_mqps']:9.1f} | "
          f"{x['range_mqps']:9.1f} {y['range_mqps']:9.1f}")
