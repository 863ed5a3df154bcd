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
run(512, 27, L=500)               # 4 levels, long slices: walk_flat; one level after cleanup: warp from start
run(1024, 63, L=64, alphabet=20_000)  # 6 levels with duplicates: walk_flat, range phase 2 both paths
# owner-routed sharding kernels (route / piece sum / piece assemble) vs the numpy stand-ins
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_sharded_gloo import CpuTestBackend  # noqa: E402
cpu, gs = CpuTestBackend(16), pkg.GpuLSM(16)
k1 = synth.uniform_u32(5, 1, 2000)
k2 = np.minimum(k1.astype(np.uint64) + (synth.uniform_u32(5, 2, 2000) >> np.uint32(22)), 0xFFFFFFFF).astype(np.uint32)
k2[::7] = 0xFFFFFFFF
t1, t2 = torch.from_numpy(k1.view(np.int32).copy()), torch.from_numpy(k2.view(np.int32).copy())
pk1, pk2, ps = gs.shard_route_ranges(t1.cuda(), t2.cuda(), 3)
c1, c2, cps = cpu.route_ranges(t1, t2, 3)
assert np.array_equal(ps.cpu().numpy(), cps.numpy()) and np.array_equal(pk1.cpu().numpy(), c1.numpy())
_, _, _, perm, cnt = gs.shard_bucket(pk1, 3, vals=pk2, want_perm=True)
pc = (np.arange(pk1.numel()) % 5).astype(np.int32)
assert np.array_equal(gs.shard_piece_sum(torch.from_numpy(pc).cuda(), perm, ps, 2000).cpu().numpy(),
                      cpu.piece_sum(torch.from_numpy(pc), perm.cpu(), cps, 2000).numpy())
ch = cnt.cpu().numpy().astype(np.int64)
cs = np.concatenate([[0], np.cumsum(ch)])
offs = np.zeros(pk1.numel(), np.int64)
blen = np.zeros(3, np.int64)
for c in range(3):
    seg = pc[cs[c]:cs[c + 1]].astype(np.int64)
    if len(seg):
        offs[cs[c]:cs[c + 1]] = 7 + np.concatenate([[0], np.cumsum(seg)[:-1]])
    blen[c] = seg.sum()
kin = np.arange(int(blen.sum()), dtype=np.int32)
args = [torch.from_numpy(offs), torch.from_numpy(blen), cnt.cpu(), 3, perm.cpu(), cps, 2000,
        torch.from_numpy(kin), torch.from_numpy(kin)]
eo, ek, _ = cpu.piece_assemble(*args)
o_, k_, _ = gs.shard_piece_assemble(*[a.cuda() if isinstance(a, torch.Tensor) else a for a in args])
assert np.array_equal(o_.cpu().numpy(), eo.numpy()) and np.array_equal(k_.cpu().numpy(), ek.numpy())
if os.environ.get("SAN_BIG"):
    run(1_100_000, 2)                 # above one wave: the two-level MSD + rank sort
g = pkg.GpuLSM(256)
k, v, d = synth.updates(3, 0, 2000, delete_frac4=1, alphabet=700)
g.bulk_build(to_device(k), to_device(v), to_device(d)); g.sync()
print("sanitize run ok")
