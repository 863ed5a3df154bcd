"""GPU parity at the sizes and launch configurations bench.py times.

The parity tests of test_gpu_parity.py use small query batches (<= 50 K), so
the query kernels never loop over many CTA rounds there. These tests run the
kernels exactly as bench.py does -- C3 (BASELINE configs[2]): b = 2^20, 64
mixed batches, 2^24 lookups / counts / ranges at L = 8, cleanup, the same
queries again -- and compare with the oracle:

* levels bit-exact vs S1 (the structural oracle, fed every update) after
  r = 64 and after the cleanup;
* lookups / counts / ranges vs O1 restricted to a key sub-range (keys never
  interact, so O1 fed only the updates whose key lies in
  [lo, hi) answers every query inside [lo, hi) exactly). The bench's own
  2^24 queries are checked wherever the oracle can vouch for them (query
  inside the sub-range), and properties that hold at any size are checked
  for all of them (offsets = exclusive scan of the counts, count ==
  len(range)); a further 2^22 ranges / counts / lookups aimed inside the
  sub-range are compared element by element (many 1024-query blocks per CTA,
  look-back across rounds);
* count / range on more than 8 occupied levels (the generic kernels) vs the
  full O1.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")

import paper_1707_05354_b200 as pkg  # noqa: E402
from paper_1707_05354_b200 import to_device, to_numpy_u32  # noqa: E402

B = 1 << 20
R = 64
NQ = 1 << 24
SEED = synth.SEED_BASE + 2  # bench.py's C3 seed
LO, HI = 5 << 25, 6 << 25   # 1/64 of the key domain


def _levels_equal(g, s1, where):
    assert g.r == s1.r, where
    for i in range(max(g.r.bit_length(), s1.num_levels())):
        gk, gv = g.level(i)
        gk, gv = to_numpy_u32(gk), to_numpy_u32(gv)
        sk, sv = s1.level(i) if i < s1.num_levels() else (np.zeros(0, np.uint32),) * 2
        assert len(gk) == len(sk), f"{where} level {i}: {len(gk)} vs {len(sk)}"
        if not np.array_equal(gk, sk):
            bad = np.nonzero(gk != sk)[0]
            raise AssertionError(f"{where} level {i} keys differ at {bad[:8]}")
        assert np.array_equal(gv, sv), f"{where} level {i} vals differ"
        del gk, gv, sk, sv


def _inside(k1, k2):
    return (k1 >= LO) & (k2 < HI) & (k1 <= k2)


def _check_bench_queries(g, o1, q, k1, k2, tag):
    """The bench's 2^24 queries, in the bench's launch configuration."""
    dq, dk1, dk2 = to_device(q), to_device(k1), to_device(k2)
    gv, gf = g.lookup(dq)
    gv, gf = to_numpy_u32(gv), gf.cpu().numpy()
    sel = (q >= LO) & (q < HI)
    ov, of = o1.lookup(q[sel])
    assert np.array_equal(gf[sel], of), tag
    assert np.array_equal(gv[sel], ov), tag
    gc = to_numpy_u32(g.count(dk1, dk2))
    ins = _inside(k1, k2)
    assert np.array_equal(gc[ins], o1.count(k1[ins], k2[ins])), tag
    off, ks, vs = g.range(dk1, dk2)
    off = off.cpu().numpy().astype(np.uint64)
    # offsets of ALL 2^24 queries: exclusive scan of the counts (any size)
    assert off[0] == 0
    assert np.array_equal(np.diff(off), gc.astype(np.uint64)), tag
    ks, vs = to_numpy_u32(ks), to_numpy_u32(vs)
    assert len(ks) == int(off[-1])
    # pairs of the queries inside the sub-range, at their offsets
    idx = np.nonzero(ins)[0]
    ooff, oks, ovs = o1.range(k1[idx], k2[idx])
    lens = np.diff(ooff).astype(np.int64)
    pos = np.repeat(off[idx].astype(np.int64), lens) + (
        np.arange(int(lens.sum())) - np.repeat(ooff[:-1].astype(np.int64), lens))
    assert np.array_equal(ks[pos], oks), tag
    assert np.array_equal(vs[pos], ovs), tag
    # every returned pair lies in its query's interval, ascending (any size)
    qid = np.repeat(np.arange(NQ), gc.astype(np.int64))
    assert np.all((ks >= k1[qid]) & (ks <= k2[qid])), tag
    same = qid[1:] == qid[:-1]
    assert np.all(ks[1:][same] > ks[:-1][same]), tag


def _check_dense_queries(g, o1, n_res, tag):
    """2^22 ranges / counts / lookups all inside the sub-range: every output
    compared with O1 (4096 range blocks, many per CTA)."""
    nq = 1 << 22
    rng = np.random.default_rng(3)
    w = max(1, round(8 * synth.D / n_res))
    k1 = rng.integers(LO, HI - w, nq).astype(np.uint32)
    k2 = (k1 + w - 1).astype(np.uint32)
    gc = to_numpy_u32(g.count(to_device(k1), to_device(k2)))
    assert np.array_equal(gc, o1.count(k1, k2)), tag
    off, ks, vs = g.range(to_device(k1), to_device(k2))
    ooff, oks, ovs = o1.range(k1, k2)
    assert np.array_equal(off.cpu().numpy().astype(np.uint64), ooff), tag
    assert np.array_equal(to_numpy_u32(ks), oks) and np.array_equal(to_numpy_u32(vs), ovs), tag
    live = o1.items()[0]
    q = np.concatenate([live[rng.integers(0, len(live), nq // 2)],
                        rng.integers(LO, HI, nq // 2).astype(np.uint32)])
    gv, gf = g.lookup(to_device(q))
    ov, of = o1.lookup(q)
    assert np.array_equal(gf.cpu().numpy(), of), tag
    assert np.array_equal(to_numpy_u32(gv), ov), tag


def test_c3_bench_configuration():
    g = pkg.GpuLSM(B, reserve_batches=R)
    s1 = oracle.ShadowLSM(B)
    o1 = oracle.OracleDict(B)
    for j in range(R):
        k, v, d = synth.updates(SEED, j * B, B, delete_frac4=1)
        g.update(to_device(k), to_device(v), to_device(d))
        s1.update(k, v, d)
        sel = (k >= LO) & (k < HI)
        o1.apply_batch(k[sel], v[sel], d[sel])
    g.sync()
    _levels_equal(g, s1, "C3 r=64")
    q = synth.lookup_queries(SEED, NQ, R * B)
    k1, k2 = synth.range_queries(SEED, NQ, R * B, 8)
    _check_bench_queries(g, o1, q, k1, k2, "C3 before cleanup")
    _check_dense_queries(g, o1, R * B, "C3 dense before cleanup")
    g.cleanup()
    s1.cleanup()
    o1.cleanup()
    _levels_equal(g, s1, "C3 after cleanup")
    del s1
    _check_bench_queries(g, o1, q, k1, k2, "C3 after cleanup")
    _check_dense_queries(g, o1, R * B, "C3 dense after cleanup")


@pytest.mark.parametrize("r", [511, 1023])
def test_count_range_more_than_8_levels(r):
    # popcount(r) = 9 / 10 occupied levels: the generic count / range kernels
    # (level state in local memory, dynamically claimed 32-query tasks with a
    # per-task look-back), vs the full O1; enough queries for many rounds
    b = 64
    seed = synth.SEED_BASE + 120 + r % 7
    g = pkg.GpuLSM(b)
    o1 = oracle.OracleDict(b)
    alpha = 40_000
    k, v, d = synth.updates(seed, 0, r * b, delete_frac4=1, alphabet=alpha)
    g.update_batches(to_device(k), to_device(v), to_device(d))
    for j in range(r):
        sl = slice(j * b, (j + 1) * b)
        o1.apply_batch(k[sl], v[sl], d[sl])
    assert g.r == r and bin(r).count("1") > 8
    for L in (8, 200):
        k1, k2 = synth.range_queries(seed + L, 400_000, r * b, L, domain=alpha + 2)
        gc = to_numpy_u32(g.count(to_device(k1), to_device(k2)))
        assert np.array_equal(gc, o1.count(k1, k2)), L
        off, ks, vs = g.range(to_device(k1), to_device(k2))
        ooff, oks, ovs = o1.range(k1, k2)
        assert np.array_equal(off.cpu().numpy().astype(np.uint64), ooff), L
        assert np.array_equal(to_numpy_u32(ks), oks), L
        assert np.array_equal(to_numpy_u32(vs), ovs), L
    q = synth.lookup_queries(seed, 400_000, r * b, alphabet=alpha)
    gv, gf = g.lookup(to_device(q))
    ov, of = o1.lookup(q)
    assert np.array_equal(gf.cpu().numpy(), of) and np.array_equal(to_numpy_u32(gv), ov)


@pytest.mark.parametrize("r", [1, 7])
def test_queries_many_rounds_exact(r):
    # 2^21 queries against a full O1 on 1 and 3 levels: lookup / count grid-
    # stride loops and range_block's multi-round block claim + look-back,
    # every output compared
    b = 1 << 16
    seed = synth.SEED_BASE + 130 + r
    g = pkg.GpuLSM(b)
    o1 = oracle.OracleDict(b)
    for j in range(r):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=1)
        g.update(to_device(k), to_device(v), to_device(d))
        o1.apply_batch(k, v, d)
    nq = 1 << 21
    for L in (8, 64):
        k1, k2 = synth.range_queries(seed + L, nq, r * b, L)
        gc = to_numpy_u32(g.count(to_device(k1), to_device(k2)))
        assert np.array_equal(gc, o1.count(k1, k2)), L
        off, ks, vs = g.range(to_device(k1), to_device(k2))
        ooff, oks, ovs = o1.range(k1, k2)
        assert np.array_equal(off.cpu().numpy().astype(np.uint64), ooff), L
        assert np.array_equal(to_numpy_u32(ks), oks) and np.array_equal(to_numpy_u32(vs), ovs), L
    q = synth.lookup_queries(seed, nq, r * b)
    gv, gf = g.lookup(to_device(q))
    ov, of = o1.lookup(q)
    assert np.array_equal(gf.cpu().numpy(), of) and np.array_equal(to_numpy_u32(gv), ov)


def test_concurrent_queries_two_streams():
    # queries on two streams at once (include/gpulsm.h: per-call scratch, the
    # index finalize ordered through an event): both results exact vs O1
    b = 1 << 16
    seed = synth.SEED_BASE + 140
    g = pkg.GpuLSM(b)
    o1 = oracle.OracleDict(b)
    for j in range(5):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=1)
        g.update(to_device(k), to_device(v), to_device(d))
        o1.apply_batch(k, v, d)
    torch.cuda.synchronize()
    import threading
    s_a, s_b = torch.cuda.Stream(), torch.cuda.Stream()
    k1a, k2a = synth.range_queries(seed + 1, 300_000, 5 * b, 8)
    k1b, k2b = synth.range_queries(seed + 2, 300_000, 5 * b, 64)
    jobs = {"a": (to_device(k1a), to_device(k2a), s_a), "b": (to_device(k1b), to_device(k2b), s_b)}
    torch.cuda.synchronize()
    out, errs = {}, []

    def run(name):
        d1, d2, st = jobs[name]
        try:
            for _ in range(3):  # several calls each, overlapping in time
                out[name] = (g.range(d1, d2, stream=st), g.count(d1, d2, stream=st))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=run, args=(n,)) for n in ("a", "b")]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    for name, k1, k2 in (("a", k1a, k2a), ("b", k1b, k2b)):
        (off, ks, vs), c = out[name]
        ooff, oks, ovs = o1.range(k1, k2)
        assert np.array_equal(off.cpu().numpy().astype(np.uint64), ooff)
        assert np.array_equal(to_numpy_u32(ks), oks) and np.array_equal(to_numpy_u32(vs), ovs)
        assert np.array_equal(to_numpy_u32(c), o1.count(k1, k2))
