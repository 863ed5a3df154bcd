"""Lookup rate vs the number of occupied levels (b = 2^20 mixed batches, r in
{3, 7, 15, 31, 63, 127}, 2^24 lookups, 50 % hits), CUDA-event timing (median of
3 after a warm-up); a sampled check against O1 on the key sub-range.

    python scripts/lookup_levels.py [--rs 3,7,15]
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

ap = argparse.ArgumentParser()
ap.add_argument("--rs", default="3,7,15,31,63,127")
a = ap.parse_args()
b = 1 << 20
seed = synth.SEED_BASE + 5
RS = [int(x) for x in a.rs.split(",")]
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
lsm = pkg.GpuLSM(b, reserve_batches=max(RS))
stream = torch.cuda.current_stream()
nq = 1 << 24
r = 0
for target in RS:
    while r < target:
        lsm.update(*synth.updates_t(seed, r * b, b, delete_frac4=1, device=dev))
        r += 1
    q = synth.lookup_queries_t(seed, nq, r * b, device=dev)
    vals = torch.empty(nq, dtype=torch.int32, device=dev)
    found = torch.empty(nq, dtype=torch.uint8, device=dev)
    lsm.lookup_into(q, vals, found)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lsm.lookup_into(q, vals, found)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    print(json.dumps({"r": r, "levels": lsm.query_levels, "nq": nq, "lookup_ms": ms,
                      "lookup_mqps": nq / (ms * 1e-3) / 1e6,
                      "hit_frac": float(found.float().mean().item())}), flush=True)
