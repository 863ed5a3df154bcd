"""One C4 point for ncu captures (not a bench): b = 2^20 insert-only batches up
to r, then count and range at expected length L.

    python scripts/prof_c4.py [--r 127] [--L 1024]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1707_05354_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--r", type=int, default=127)
ap.add_argument("--L", type=int, default=1024)
a = ap.parse_args()
b = 1 << 20
seed = synth.SEED_BASE + 3
dev = torch.device("cuda", 0)
lsm = pkg.GpuLSM(b, reserve_batches=a.r)
for j in range(a.r):
    lsm.update(*synth.updates_t(seed, j * b, b, delete_frac4=0, device=dev))
n = a.r * b
nq = min(1 << 24, (1 << 27) // a.L)
k1, k2 = synth.range_queries_t(seed + a.L, nq, n, a.L, device=dev)
cnt = lsm.count(k1, k2)
off, rk, rv = lsm.range(k1, k2)
torch.cuda.synchronize()
print("levels", lsm.query_levels, "pairs", int(off[-1].item()))
