"""Small end-to-end run of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck). Exits non-zero on any parity failure."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import oracle
import synth
import paper_1707_05354_b200 as pkg
from paper_1707_05354_b200 import to_device, to_numpy_u32

def run(b, nb, sa=False, alphabet=None, frac4=1, multi=False, L=8):
    g = pkg.GpuLSM(b, sa=sa)
    o = oracle.OracleDict(b)
    seed = synth.SEED_BASE + b % 97
    if multi:
        k, v, d = synth.updates(seed, 0, nb * b - 3, delete_frac4=frac4, alphabet=alphabet)
        g.update_batches(to_device(k), to_device(v), to_device(d))
        for j in range(nb):
            sl = slice(j * b, min(len(k), (j + 1) * b)); o.apply_batch(k[sl], v[sl], d[sl])
    else:
        for j in range(nb):
            k, v, d = synth.updates(seed, j * b, b, delete_frac4=frac4, alphabet=alphabet)
            g.update(to_device(k), to_device(v), to_device(d)); o.apply_batch(k, v, d)
    n = nb * b
    q = synth.lookup_queries(seed, 3000, n, alphabet)
    k1, k2 = synth.range_queries(seed, 500, n, L, domain=alphabet or synth.D)
    for phase in range(2):
        gv, gf = g.lookup(to_device(q)); ov, of = o.lookup(q)
        assert np.array_equal(gf.cpu().numpy(), of) and np.array_equal(to_numpy_u32(gv), ov)
        assert np.array_equal(to_numpy_u32(g.count(to_device(k1), to_device(k2))), o.count(k1, k2))
        off, ks, vs = g.range(to_device(k1), to_device(k2)); ooff, oks, ovs = o.range(k1, k2)
        assert np.array_equal(to_numpy_u32(ks), oks) and np.array_equal(to_numpy_u32(vs), ovs)
        for fn in ("successor", "predecessor"):
            gk, gvv, gff = getattr(g, fn)(to_device(q)); ek, ev, ef = getattr(o, fn)(q)
            assert np.array_equal(to_numpy_u32(gk), ek) and np.array_equal(gff.cpu().numpy(), ef)
        g.cleanup(); o.cleanup()
    torch.cuda.synchronize()

run(100, 13)                      # odd b: misaligned views after cleanup
run(4096, 9, alphabet=5000)       # small-sort path, duplicates
run(40_000, 5)                    # MSD + bucket path, multi-level
run(64, 9, sa=True)               # GPU SA
run(1000, 7, multi=True)          # multi-batch insertion
run(8192, 4, L=2000)              # one level, long slices: warp-cooperative walk
run(20_000, 3, alphabet=3000)     # oversized bucket: regather + chunked LSD
if os.environ.get("SAN_BIG"):
    run(1_100_000, 2)                 # above one wave: the two-level MSD + rank sort
g = pkg.GpuLSM(256)
k, v, d = synth.updates(3, 0, 2000, delete_frac4=1, alphabet=700)
g.bulk_build(to_device(k), to_device(v), to_device(d)); g.sync()
print("sanitize run ok")
