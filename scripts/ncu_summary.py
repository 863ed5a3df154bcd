"""Summarise ncu outputs into profiles/ (run here, after gpurun brings them back).

    python scripts/ncu_summary.py --launches gpurun_out/launches.csv \
        --reps gpurun_out/prof_*.ncu-rep --round r01

Writes profiles/<round>_launches_summary.txt (per-kernel share of device time
from the launch list), profiles/<round>_ncu_full_summary.txt (key metrics and
top stall reasons per captured launch) and profiles/ncu_traffic.json (DRAM
bytes per launch per kernel, read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import glob
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUL = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TMUL = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}

CLASS = [("onesweep", "sort_pass"), ("bucket_sort", "sort_pass"), ("small_sort", "sort_pass"),
         ("msd_scatter", "sort_pass"), ("bucket_rank", "sort_pass"),
         ("sort_hist", "sort_hist"), ("merge_kernel", "merge"),
         ("lookup_kernel", "lookup"), ("range_block", "range"),
         ("count_kernel", "count"), ("range_kernel", "range"),
         ("build_f1", "other"), ("finalize_index", "other"),
         ("scan_", "scan"), ("cleanup_", "cleanup"), ("fill_placebo", "cleanup"),
         ("bucket_", "other"), ("scatter_back", "other"), ("clip_kernel", "other"),
         ("sum_parts", "other")]


def kclass(name):
    for pat, c in CLASS:
        if pat in name:
            return c
    return "other"


def short(name):
    return name.split("(")[0].replace("void ", "").split("::")[-1]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                  "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = per.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * (TMUL.get(r[ui], 1.0) if "time" in r[mi] else MUL.get(r[ui], 1.0))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        a = agg[short(d["name"])]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    return agg


def full(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        g = lambda h: r[hdr.index(h)] if h in hdr else None  # noqa: E731
        u = lambda h: units[hdr.index(h)] if h in hdr else ""  # noqa: E731
        t = float(g("gpu__time_duration.sum")) * TMUL.get(u("gpu__time_duration.sum"), 1.0)
        rd = float(g("dram__bytes_read.sum")) * MUL.get(u("dram__bytes_read.sum"), 1.0)
        wr = float(g("dram__bytes_write.sum")) * MUL.get(u("dram__bytes_write.sum"), 1.0)
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        res.append({
            "kernel": short(g("Kernel Name")), "class": kclass(g("Kernel Name")),
            "grid": g("launch__grid_size"), "block": g("launch__block_size"),
            "regs": g("launch__registers_per_thread"),
            "time_us": t, "dram_read_bytes": rd, "dram_write_bytes": wr,
            "dram_GBps": (rd + wr) / (t * 1e-6) / 1e9 if t else None,
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "l2_throughput_pct": g("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "smem_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "smem_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "l1_hit_pct": g("l1tex__t_sector_hit_rate.pct"),
            "l2_hit_pct": g("lts__t_sector_hit_rate.pct"),
            "top_stalls": [(n, round(v, 2)) for v, n in sorted(stalls, reverse=True)[:5]],
            "rep": os.path.basename(rep),
        })
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--reps", nargs="*", default=[])
    ap.add_argument("--round", default="r01")
    ap.add_argument("--units", default="{}", help="json: class -> units per captured launch")
    ap.add_argument("--outdir", default=os.path.join(ROOT, "profiles"))
    a = ap.parse_args()
    prof = a.outdir
    os.makedirs(prof, exist_ok=True)
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v[1] for v in agg.values())
        lines = [f"# ncu launch list ({a.launches}); device time per kernel, cold-cache and serialised",
                 f"# total {tot / 1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches",
                 f"{'kernel':34s} {'launches':>8s} {'total_ms':>10s} {'share':>7s} {'avg_us':>9s}"]
        for n, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"{n:34s} {v[0]:8d} {v[1] / 1e3:10.3f} {100 * v[1] / tot:6.1f}% {v[1] / v[0]:9.2f}")
        open(os.path.join(prof, f"{a.round}_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    reps = [r for pat in a.reps for r in glob.glob(pat)]
    if reps:
        allres = []
        for r in reps:
            allres.extend(full(r))
        lines = []
        for x in allres:
            lines.append(f"{x['kernel']} [{x['class']}] grid={x['grid']} block={x['block']} regs={x['regs']} "
                         f"t={x['time_us']:.2f}us dram={(x['dram_read_bytes'] + x['dram_write_bytes']) / 1e6:.2f}MB "
                         f"({x['dram_GBps'] or 0:.0f} GB/s) issue={x['issue_active_pct']}% "
                         f"warps={x['warps_active_pct']}% l2={x['l2_throughput_pct']}% l2hit={x['l2_hit_pct']}% "
                         f"smem_wf={x['smem_wavefronts']} smem_conf={x['smem_bank_conflicts']} stalls={x['top_stalls']} "
                         f"[{x['rep']}]")
        open(os.path.join(prof, f"{a.round}_ncu_full_summary.txt"), "w").write("\n".join(lines) + "\n")
        json.dump(allres, open(os.path.join(prof, f"{a.round}_ncu_full.json"), "w"), indent=1)
        print("\n".join(lines))
        # traffic per class: DRAM bytes per launch averaged over the captured
        # launches of the class's largest-traffic report (range = count pass +
        # write pass, both captured from one range call)
        units = json.loads(a.units)
        by = collections.defaultdict(list)
        for x in allres:
            by[(x["class"], x["rep"])].append(x)
        traffic = {}
        for (c, rep), xs in by.items():
            b = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in xs) / len(xs)
            if c not in traffic or b > traffic[c]["dram_bytes_per_launch"]:
                traffic[c] = {"dram_bytes_per_launch": b, "launches_captured": len(xs),
                              "time_us": sum(x["time_us"] for x in xs) / len(xs),
                              "kernel": "+".join(sorted({x["kernel"] for x in xs})),
                              "rep": rep, "units_per_launch": units.get(c)}
        json.dump(traffic, open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
