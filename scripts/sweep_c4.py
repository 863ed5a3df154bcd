"""C4 query sweep (BASELINE.json configs[3]): b = 2^20 insert-only
batches, r in {96, 112, 120, 124, 126, 127, 128} (1..7 occupied levels, n =
0.75..1.0 x 2^27), count and range at expected range lengths L = 8..1024 with
nq = min(2^24, 2^27 / L). CUDA-event timing (median of 3 after a warm-up), and
per row the measured mean valid pairs per query; sum(count) == len(range) is
checked on every row (count == length of range).

    python scripts/sweep_c4.py [--out profiles/r01_sweep_c4.json] [--quick]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1707_05354_b200 as pkg  # noqa: E402
from paper_1707_05354_b200 import to_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--quick", action="store_true", help="r in {96, 127} and L in {8, 128, 1024}")
ap.add_argument("--rs", default=None, help="comma-separated r values (overrides the default set)")
ap.add_argument("--ls", default=None, help="comma-separated L values")
a = ap.parse_args()

b = 1 << 20
RS = [96, 127] if a.quick else [96, 112, 120, 124, 126, 127, 128]
LS = [8, 128, 1024] if a.quick else [8, 16, 32, 64, 128, 256, 512, 1024]
if a.rs:
    RS = [int(x) for x in a.rs.split(",")]
if a.ls:
    LS = [int(x) for x in a.ls.split(",")]
seed = synth.SEED_BASE + 3
torch.cuda.set_device(0)
lsm = pkg.GpuLSM(b, reserve_batches=max(RS))
stream = torch.cuda.current_stream()


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


rows = []
r = 0
for target in RS:
    while r < target:
        k, v, d = synth.updates(seed, r * b, b, delete_frac4=0)
        lsm.update(to_device(k), to_device(v), to_device(d))
        r += 1
    torch.cuda.synchronize()
    levels = bin(r).count("1")
    n = r * b
    for L in LS:
        nq = min(1 << 24, (1 << 27) // L)
        k1, k2 = synth.range_queries(seed + L, nq, n, L)
        k1, k2 = to_device(k1), to_device(k2)
        cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
        t_count = timed(lambda: lsm.count_into(k1, k2, cnt))
        total_count = int(cnt.to(torch.int64).sum().item())
        cap = max(16, int(total_count * 1.05) + 16)
        off = torch.empty(nq + 1, dtype=torch.int64, device="cuda")
        rk = torch.empty(cap, dtype=torch.int32, device="cuda")
        rv = torch.empty(cap, dtype=torch.int32, device="cuda")
        got = []
        t_range = timed(lambda: got.append(lsm.range_into(k1, k2, off, rk, rv)))
        assert got[-1] == total_count, (r, L, got[-1], total_count)  # count == len(range)
        row = {"r": r, "levels": levels, "n": n, "L": L, "nq": nq,
               "count_ms": t_count, "count_mqps": nq / (t_count * 1e-3) / 1e6,
               "range_ms": t_range, "range_mqps": nq / (t_range * 1e-3) / 1e6,
               "pairs_per_query": total_count / nq,
               "range_out_GBps": total_count * 8 / (t_range * 1e-3) / 1e9}
        rows.append(row)
        print(json.dumps(row), flush=True)
if a.out:
    with open(a.out, "w") as f:
        json.dump({"config": "C4: b=2^20 insert-only, r in %s, L in %s" % (RS, LS), "rows": rows}, f,
                  indent=1)
