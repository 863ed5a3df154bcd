"""One C3 cycle for ncu captures (not a bench): 64 mixed batches of 2^20, then
lookup/count/range on r = 64, cleanup, lookup/count/range again.

    python scripts/prof_step.py [--batches 64] [--nq 16777216] [--b 1048576]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1707_05354_b200 as pkg  # noqa: E402
from paper_1707_05354_b200 import to_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=1 << 20)
ap.add_argument("--batches", type=int, default=64)
ap.add_argument("--nq", type=int, default=1 << 24)
ap.add_argument("--L", type=float, default=8)
ap.add_argument("--no-cleanup", action="store_true")
a = ap.parse_args()

seed = synth.SEED_BASE + 2
b = a.b
lsm = pkg.GpuLSM(b, reserve_batches=a.batches)
for j in range(a.batches):
    k, v, d = synth.updates(seed, j * b, b, delete_frac4=1)
    lsm.update(to_device(k), to_device(v), to_device(d))
torch.cuda.synchronize()
n = a.batches * b
q = to_device(synth.lookup_queries(seed, a.nq, n))
k1, k2 = synth.range_queries(seed, a.nq, n, a.L)
k1, k2 = to_device(k1), to_device(k2)
vals, found = lsm.lookup(q)
cnt = lsm.count(k1, k2)
off, rk, rv = lsm.range(k1, k2)
if not a.no_cleanup:
    lsm.cleanup()
    vals, found = lsm.lookup(q)
    cnt = lsm.count(k1, k2)
    off, rk, rv = lsm.range(k1, k2)
torch.cuda.synchronize()
print("done r=", lsm.r, "launches=", lsm.launch_count)
