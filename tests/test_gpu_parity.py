"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Structure: level key/value arrays bit-exact vs S1 after every mutation.
Queries: lookup / count / range results exactly equal to O1 (range compared
per query as the sorted pair list, which is unique). All integer work, so
the tolerance is zero (BASELINE.json north_star).
"""
import numpy as np
import pytest

import oracle
import synth
from tests import lsm_script

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_1707_05354_b200 as pkg  # noqa: E402
from paper_1707_05354_b200 import to_device, to_numpy_u32  # noqa: E402


class GpuAdapter:
    def __init__(self, b):
        self.lsm = pkg.GpuLSM(b)

    def update(self, k, v, d):
        self.lsm.update(to_device(k), to_device(v), to_device(d.astype(np.uint8)))

    def lookup(self, q):
        v, f = self.lsm.lookup(to_device(q))
        return to_numpy_u32(v), f.cpu().numpy()

    def count(self, k1, k2):
        return to_numpy_u32(self.lsm.count(to_device(k1), to_device(k2)))

    def successor(self, q):
        k, v, f = self.lsm.successor(to_device(q))
        return to_numpy_u32(k), to_numpy_u32(v), f.cpu().numpy()

    def predecessor(self, q):
        k, v, f = self.lsm.predecessor(to_device(q))
        return to_numpy_u32(k), to_numpy_u32(v), f.cpu().numpy()

    def range(self, k1, k2):
        off, ks, vs = self.lsm.range(to_device(k1), to_device(k2))
        return off.cpu().numpy().astype(np.uint64), to_numpy_u32(ks), to_numpy_u32(vs)

    def cleanup(self):
        self.lsm.cleanup()

    @property
    def r(self):
        return self.lsm.r

    def level(self, i):
        k, v = self.lsm.level(i)
        return to_numpy_u32(k), to_numpy_u32(v)

    def num_levels(self):
        return max(self.r.bit_length(), 1)


def assert_levels_equal(gpu, s1, where=""):
    assert gpu.r == s1.r, where
    for i in range(max(gpu.r.bit_length(), s1.num_levels())):
        gk, gv = gpu.level(i)
        sk, sv = s1.level(i) if i < s1.num_levels() else (np.zeros(0, np.uint32),) * 2
        assert len(gk) == len(sk), f"{where} level {i}: {len(gk)} vs {len(sk)}"
        if not np.array_equal(gk, sk):
            bad = np.nonzero(gk != sk)[0]
            raise AssertionError(f"{where} level {i} keys differ at {bad[:10]} "
                                 f"gpu={gk[bad[:10]]} s1={sk[bad[:10]]}")
        assert np.array_equal(gv, sv), f"{where} level {i} vals differ"


def assert_queries_equal(gpu, o1, lookups, k1, k2, where=""):
    gv, gf = gpu.lookup(lookups)
    ov, of = o1.lookup(lookups)
    assert np.array_equal(gf, of), f"{where} lookup found mismatch"
    assert np.array_equal(gv, ov), f"{where} lookup value mismatch"
    gc = gpu.count(k1, k2)
    oc = o1.count(k1, k2)
    assert np.array_equal(gc, oc), f"{where} count mismatch at {np.nonzero(gc != oc)[0][:10]}"
    goff, gk, gvv = gpu.range(k1, k2)
    ooff, ok, ovv = o1.range(k1, k2)
    assert np.array_equal(goff, ooff), f"{where} range offsets mismatch"
    assert np.array_equal(gk, ok) and np.array_equal(gvv, ovv), f"{where} range pairs mismatch"
    assert np.array_equal(np.diff(goff).astype(np.uint32), gc)  # count == len(range)
    assert_order_equal(gpu, o1, lookups, where)


def assert_order_equal(gpu, o1, q, where=""):
    """N3 successor / predecessor (R23), exact vs O1."""
    for name in ("successor", "predecessor"):
        gk, gv, gf = getattr(gpu, name)(q)
        ok, ov, of = getattr(o1, name)(q)
        bad = np.nonzero((gk != ok) | (gv != ov) | (gf != of))[0]
        assert len(bad) == 0, (f"{where} {name} mismatch at {bad[:8]}: q={q[bad[:8]]} "
                               f"gpu={gk[bad[:8]]},{gf[bad[:8]]} o1={ok[bad[:8]]},{of[bad[:8]]}")


@pytest.mark.parametrize("path", lsm_script.golden_files(), ids=lambda p: p.split("/")[-1])
def test_golden_scripts_gpu(path):
    lsm_script.run(path, GpuAdapter)


def _run_schedule(b, nbatch, seed, frac4=1, alphabet=None, nlook=2000, nrange=300,
                  Ls=(8, 64), cleanup_every=None, check_levels=True):
    g = GpuAdapter(b)
    s1 = oracle.ShadowLSM(b)
    o1 = oracle.OracleDict(b)
    dom = synth.D if alphabet is None else alphabet + 2
    for j in range(nbatch):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=frac4, alphabet=alphabet)
        g.update(k, v, d)
        s1.update(k, v, d)
        o1.apply_batch(k, v, d)
        if check_levels:
            assert_levels_equal(g, s1, f"b={b} batch {j}")
        q = synth.lookup_queries(seed + j, nlook, (j + 1) * b, alphabet)
        L = Ls[j % len(Ls)]
        k1, k2 = synth.range_queries(seed + j, nrange, (j + 1) * b, L, domain=dom)
        assert_queries_equal(g, o1, q, k1, k2, f"b={b} batch {j}")
        if cleanup_every and (j + 1) % cleanup_every == 0:
            g.cleanup()
            s1.cleanup()
            o1.cleanup()
            assert_levels_equal(g, s1, f"b={b} cleanup after {j}")
            assert_queries_equal(g, o1, q, k1, k2, f"b={b} after cleanup {j}")
    return g, s1, o1


def test_config_c1():
    # BASELINE.json configs[0]: b=1024, r=15 batches, 75% insert / 25% delete,
    # 10^4 lookups + 10^3 count/range queries; then cleanup and repeat.
    b = 1024
    g, s1, o1 = _run_schedule(b, 15, synth.SEED_BASE + 0, frac4=1, nlook=10_000, nrange=1000)
    g.cleanup()
    s1.cleanup()
    o1.cleanup()
    assert_levels_equal(g, s1, "C1 cleanup")
    q = synth.lookup_queries(synth.SEED_BASE, 10_000, 15 * b)
    k1, k2 = synth.range_queries(synth.SEED_BASE, 1000, 15 * b, 8)
    assert_queries_equal(g, o1, q, k1, k2, "C1 after cleanup")
    # idempotence
    g.cleanup()
    s1.cleanup()
    assert_levels_equal(g, s1, "C1 second cleanup")


def test_config_c1_duplicates():
    # C1-dup: keys mod 4096 force duplicates, in-batch insert+delete, re-inserts
    _run_schedule(1024, 15, synth.SEED_BASE + 10, frac4=1, alphabet=4096, nlook=5000,
                  nrange=500, cleanup_every=5)


@pytest.mark.parametrize("b", [1, 2, 3, 5, 33, 100, 4095, 4096, 4097, 10_000])
def test_ragged_batch_sizes(b):
    nb = 9 if b < 5000 else 5
    _run_schedule(b, nb, 77 + b, frac4=2, alphabet=3 * b + 7, nlook=500, nrange=100,
                  cleanup_every=4)


@pytest.mark.parametrize("b", [1 << 16, (1 << 17) + 123])
def test_multi_tile_sort_and_merge(b):
    # several sort tiles (7168) with a ragged tail; merges of 2b and 4b over
    # many merge tiles; uniform 31-bit keys
    _run_schedule(b, 4, 4242, frac4=1, nlook=20_000, nrange=2000)


def test_multi_wave_sort():
    # b > 148 sort tiles: the two-level MSD + rank sort
    _run_schedule((1 << 21) + 4097, 3, 99, frac4=1, nlook=20_000, nrange=1000)


def test_skewed_keys_bucket_overflow():
    # keys < 3000: every key variable has top digit 0, so the MSD pass puts
    # the whole batch into one bucket larger than shared memory: the chunked
    # fallback must still be exact, and later batches switch to 4-pass LSD
    _run_schedule(50_000, 5, 123, frac4=1, alphabet=3000, nlook=3000, nrange=300)


def _run_custom_keys(b, nbatch, seed, keyfn):
    """Mixed batches whose keys are keyfn(h) of the seeded hash stream (75%
    insert / 25% delete); levels vs S1 and queries vs O1 after every batch."""
    g = GpuAdapter(b)
    s1 = oracle.ShadowLSM(b)
    o1 = oracle.OracleDict(b)
    for j in range(nbatch):
        idx = np.arange(j * b, (j + 1) * b, dtype=np.uint64)
        k = keyfn(synth.h(seed, 0, idx), synth.h(seed, 5, idx)).astype(np.uint32)
        v = idx.astype(np.uint32)
        d = ((synth.h(seed, 1, idx) % np.uint64(4)) == 0).astype(np.uint8)
        g.update(k, v, d)
        s1.update(k, v, d)
        o1.apply_batch(k, v, d)
        assert_levels_equal(g, s1, f"custom b={b} batch {j}")
    q = k[: min(b, 5000)].copy()
    k1 = np.sort(k[:1000])
    k2 = k1 + np.uint32(1 << 20)
    assert_queries_equal(g, o1, q, k1, k2, "custom keys")


def test_sort_duplicate_keys_position_tiebreak():
    # 5000 distinct keys spread over the domain, b = 50,000: every key occurs
    # about ten times per batch (inserts and deletes), so the MSD + rank sort
    # must order equal key variables by input position (R4: first wins)
    _run_custom_keys(50_000, 3, 31, lambda h, h2: (h % np.uint64(5000)) * np.uint64(429_000))


def test_sort_skewed_bin_fallback():
    # every key of a top-digit bucket falls into one 11-bit bin (low key bits
    # < 200): bins far above kBinMax take the stable shared-memory fallback
    _run_custom_keys(30_000, 3, 32,
                     lambda h, h2: ((h % np.uint64(256)) << np.uint64(23)) | (h2 % np.uint64(200)))


@pytest.mark.parametrize("alphabet", [None, 30_000])
def test_long_ranges_single_level(alphabet):
    # one occupied level (r = 4) and ranges of ~100..10^4 resident records:
    # slices longer than the per-lane cap continue warp-cooperatively (run
    # heads across lane boundaries, the slice end inside a lane); the
    # duplicate-heavy alphabet puts long stale runs and tombstones in them
    b = 8192
    g = GpuAdapter(b)
    o1 = oracle.OracleDict(b)
    for j in range(4):
        k, v, d = synth.updates(41, j * b, b, delete_frac4=1, alphabet=alphabet)
        g.update(k, v, d)
        o1.apply_batch(k, v, d)
    assert g.r == 4
    dom = synth.D if alphabet is None else alphabet + 2
    for L in (100, 1000, 10_000):
        k1, k2 = synth.range_queries(42 + L, 300, 4 * b, L, domain=dom)
        q = synth.lookup_queries(43, 1000, 4 * b, alphabet)
        assert_queries_equal(g, o1, q, k1, k2, f"long ranges L={L}")


@pytest.mark.parametrize("r", [3, 6, 15, 27, 63, 127, 255, 511])
@pytest.mark.parametrize("alphabet", [None, 30_000])
def test_long_ranges_multi_level(r, alphabet):
    # 2..9 occupied levels and ranges of ~100..10^4 resident records: a lane's
    # walk stops after its key cap and the warp finishes the query in rounds
    # over shared memory (warp_merge_long) -- chunks cut at a common key,
    # validity against newer levels, slots from per-level valid ranks; the
    # duplicate-heavy alphabet gives stale runs longer than a chunk (the
    # one-step fallback) and tombstones; a partial last batch puts a placebo
    # run into the slices of ranges ending at 2^32-1 (R5, R8). r = 511 takes
    # the >8-level kernels.
    b = 1024
    g = GpuAdapter(b)
    o1 = oracle.OracleDict(b)
    seed = 71 + r
    for j in range(r):
        n = b if j + 1 < r else b - 77
        k, v, d = synth.updates(seed, j * b, n, delete_frac4=1, alphabet=alphabet)
        g.update(k, v, d)
        o1.apply_batch(k, v, d)
    assert g.r == r
    dom = synth.D if alphabet is None else alphabet + 2
    for L in (100, 1000, 10_000):
        k1, k2 = synth.range_queries(seed + L, 300 if L < 10_000 else 60, r * b, L, domain=dom)
        k2[::7] = 0xFFFFFFFF  # to the top of the 32-bit query space
        k1[::11] = 0
        q = synth.lookup_queries(seed, 1000, r * b, alphabet)
        assert_queries_equal(g, o1, q, k1, k2, f"r={r} long ranges L={L}")


def _tiny_schedules(b, nbatch, A, sample=None, seed=0):
    import itertools
    C = 2 * A
    total = C ** (b * nbatch)
    idx = range(total) if sample is None else np.random.default_rng(seed).choice(total, sample,
                                                                                 replace=False)
    for i in idx:
        x = int(i)
        digits = []
        for _ in range(b * nbatch):
            digits.append(x % C)
            x //= C
        yield digits


@pytest.mark.parametrize("b,nbatch,sample", [(2, 2, None), (4, 2, 1500), (2, 3, 1500), (1, 5, 800)])
def test_tiny_schedules_exhaustive_vs_o1(b, nbatch, sample):
    # every (or a seeded sample of the) schedule(s) of nbatch batches of b
    # updates over 3 keys x {insert, delete} (the shapes of the oracle's
    # exhaustive pins): levels bit-exact vs S1, and lookups of every key,
    # count / range of every interval vs O1 (one handle, cleared per schedule)
    A = 3
    g = GpuAdapter(b)
    q = np.arange(A + 1, dtype=np.uint32)
    k1 = np.array([a for a in range(A + 1) for z in range(a, A + 1)] + [2], np.uint32)
    k2 = np.array([z for a in range(A + 1) for z in range(a, A + 1)] + [1], np.uint32)
    for digits in _tiny_schedules(b, nbatch, A, sample, seed=b * 10 + nbatch):
        g.lsm.clear()
        s1 = oracle.ShadowLSM(b)
        o1 = oracle.OracleDict(b)
        for j in range(nbatch):
            part = digits[j * b:(j + 1) * b]
            keys = np.array([c // 2 for c in part], np.uint32)
            dels = np.array([c % 2 for c in part], np.uint8)
            vals = np.arange(j * b + 1, (j + 1) * b + 1, dtype=np.uint32)
            g.update(keys, vals, dels)
            s1.update(keys, vals, dels)
            o1.apply_batch(keys, vals, dels)
        assert_levels_equal(g, s1, f"schedule {digits}")
        gv, gf = g.lookup(q)
        ov, of = o1.lookup(q)
        assert np.array_equal(gf, of) and np.array_equal(gv[gf == 1], ov[of == 1]), digits
        assert np.array_equal(g.count(k1, k2), o1.count(k1, k2)), digits
        goff, gk, gvv = g.range(k1, k2)
        ooff, ok, ovv = o1.range(k1, k2)
        assert np.array_equal(goff, ooff) and np.array_equal(gk, ok) and np.array_equal(gvv, ovv), digits


def test_one_wave_boundary_sort():
    # exactly 148 tiles (largest one-wave batch) and one record more
    for b in (148 * 7168, 148 * 7168 + 1):
        _run_schedule(b, 2, 5 + b % 7, frac4=1, nlook=5000, nrange=500)


def test_partial_batches():
    b = 1000
    g = GpuAdapter(b)
    s1 = oracle.ShadowLSM(b)
    o1 = oracle.OracleDict(b)
    rng = np.random.default_rng(5)
    for j in range(12):
        n = int(rng.integers(1, b + 1))
        k, v, d = synth.updates(9, j * b, n, delete_frac4=1, alphabet=2000)
        g.update(k, v, d)
        s1.update(k, v, d)
        o1.apply_batch(k, v, d)
        assert_levels_equal(g, s1, f"partial {j}")
    q = np.arange(2002, dtype=np.uint32)
    k1, k2 = synth.range_queries(1, 200, 12 * b, 20, domain=2002)
    assert_queries_equal(g, o1, q, k1, k2, "partial")


def test_edge_queries():
    b = 64
    g = GpuAdapter(b)
    o1 = oracle.OracleDict(b)
    # queries on an empty LSM (R22)
    q = np.array([0, 1, 0x7FFFFFFE, 0x7FFFFFFF, 0xFFFFFFFF], np.uint32)
    v, f = g.lookup(q)
    assert not f.any() and np.all(v == pkg.LSM_NOT_FOUND)
    assert g.count(np.array([0], np.uint32), np.array([0xFFFFFFFF], np.uint32))[0] == 0
    off, ks, vs = g.range(np.array([0], np.uint32), np.array([0xFFFFFFFF], np.uint32))
    assert off.tolist() == [0, 0] and len(ks) == 0
    # empty query batch (nq == 0)
    e = torch.empty(0, dtype=torch.int32, device="cuda")
    vv, ff = g.lsm.lookup(e)
    assert vv.numel() == 0
    assert g.lsm.count(e, e).numel() == 0
    off, ks, vs = g.lsm.range(e, e)
    assert off.cpu().tolist() == [0]
    # max key and boundary keys; k1 > k2 (R9); a stored value 0xFFFFFFFF
    k = np.array([0, 0x7FFFFFFE, 5, 6], np.uint32)
    v = np.array([7, 8, 0xFFFFFFFF, 9], np.uint32)
    d = np.zeros(4, np.uint8)
    g.update(k, v, d)
    o1.apply_batch(k, v, d)
    q = np.array([0, 0x7FFFFFFE, 0x7FFFFFFF, 0xFFFFFFFF, 5, 6, 4], np.uint32)
    k1 = np.array([0, 6, 0x7FFFFFFE, 0, 10, 0xFFFFFFFF], np.uint32)
    k2 = np.array([0xFFFFFFFF, 5, 0xFFFFFFFF, 0x7FFFFFFE, 9, 0xFFFFFFFF], np.uint32)
    assert_queries_equal(g, o1, q, k1, k2, "edge")
    gv, gf = g.lookup(np.array([5], np.uint32))
    assert gf[0] == 1 and gv[0] == 0xFFFFFFFF


def test_out_of_domain_key_is_sticky_error():
    b = 8
    g = GpuAdapter(b)
    s1 = oracle.ShadowLSM(b)
    k = np.array([1, 0x7FFFFFFF, 2, 0xFFFFFFFF], np.uint32)
    v = np.arange(4, dtype=np.uint32)
    d = np.zeros(4, np.uint8)
    g.update(k, v, d)
    s1.update(k, v, d)
    with pytest.raises(pkg.LsmError) as ei:
        g.lsm.sync()
    assert ei.value.code == pkg.LSM_ERR_KEY_DOMAIN
    g.lsm.sync()  # cleared
    assert_levels_equal(g, s1, "domain")


def test_batch_size_errors():
    g = pkg.GpuLSM(4)
    with pytest.raises(pkg.LsmError):
        g.update(to_device(np.arange(5, dtype=np.uint32)))
    with pytest.raises(pkg.LsmError):
        g.update(to_device(np.zeros(0, dtype=np.uint32)))
    assert g.r == 0


def test_insert_delete_entry_points():
    b = 256
    g = pkg.GpuLSM(b)
    s1 = oracle.ShadowLSM(b)
    k, v, _ = synth.updates(3, 0, b, delete_frac4=0, alphabet=500)
    g.insert(to_device(k), to_device(v))
    s1.update(k, v, np.zeros(b, np.uint8))
    kd = k[: b // 2].copy()
    g.delete(to_device(kd))
    s1.update(kd, np.zeros(len(kd), np.uint32), np.ones(len(kd), np.uint8))
    ad = GpuAdapter.__new__(GpuAdapter)
    ad.lsm = g
    assert_levels_equal(ad, s1, "insert/delete")


def test_host_buffer_entry_points():
    b = 512
    g = pkg.GpuLSM(b)
    o1 = oracle.OracleDict(b)
    for j in range(6):
        k, v, d = synth.updates(21, j * b, b, delete_frac4=1, alphabet=900)
        g.update_host(k, v, d)
        o1.apply_batch(k, v, d)
    q = np.arange(902, dtype=np.uint32)
    hv, hf = g.lookup_host(q)
    ov, of = o1.lookup(q)
    assert np.array_equal(hf, of) and np.array_equal(hv, ov)


def test_host_updates_double_buffered_pinned():
    # lsm_update_host from pinned host tensors: batch j+1's copy runs on the
    # library's copy stream while batch j updates; the levels must equal those
    # of the device-buffer path (and S1) after every batch
    b = (1 << 16) + 77
    gh = pkg.GpuLSM(b)
    s1 = oracle.ShadowLSM(b)
    host = []
    for j in range(7):
        k, v, d = synth.updates(23, j * b, b, delete_frac4=1)
        host.append(tuple(torch.from_numpy(x).pin_memory() for x in (k, v, d)))
        s1.update(k, v, d)
    for j, (k, v, d) in enumerate(host):
        gh.update_host(k, v, d)
    gh.sync()
    ga = GpuAdapter(b)
    ga.lsm = gh
    assert_levels_equal(ga, s1, "pinned host updates")


def test_determinism():
    b = 3000
    imgs = []
    for _ in range(2):
        g = GpuAdapter(b)
        for j in range(7):
            k, v, d = synth.updates(99, j * b, b, delete_frac4=1, alphabet=5000)
            g.update(k, v, d)
        imgs.append([g.level(i) for i in range(3)])
    for (a, b_), (c, d_) in zip(*imgs):
        assert np.array_equal(a, c) and np.array_equal(b_, d_)


def test_launch_counter_counts_kernels():
    g = pkg.GpuLSM(4096)
    k, v, d = synth.updates(1, 0, 4096)
    n0 = g.launch_count
    g.update(to_device(k), to_device(v), to_device(d))
    # small batch (b <= 7168): one CTA sorts it in shared memory
    assert g.launch_count - n0 == 1
    g.update(to_device(k), to_device(v), to_device(d))
    assert g.launch_count - n0 == 3  # + sort + one merge
    # one-wave batch: MSD pass + per-bucket shared-memory sorts
    mid = pkg.GpuLSM(1 << 20)
    km, vm, dm = synth.updates(3, 0, 1 << 20)
    n2 = mid.launch_count
    mid.update(to_device(km), to_device(vm), to_device(dm))
    assert mid.launch_count - n2 == 2
    mid.update(to_device(km), to_device(vm), to_device(dm))
    assert mid.launch_count - n2 == 2 + 3  # sort (2) + one merge
    # multi-wave batch: two-level MSD (top-digit scatter, sub-digit scatter,
    # rank pass)
    big = pkg.GpuLSM(2_000_000)
    kb, vb, db = synth.updates(2, 0, 2_000_000)
    n1 = big.launch_count
    big.update(to_device(kb), to_device(vb), to_device(db))
    assert big.launch_count - n1 == 3


@pytest.mark.slow
def test_full_size_c3_sampled():
    """BASELINE configs[2] at full size in bench.py's launch configuration:
    b = 2^20, 64 mixed batches (n = 2^26). The oracle O1 is fed only updates
    whose key lies in a sampled sub-range (keys never interact, so the
    restriction is exact); lookups / counts / ranges inside that sub-range
    are compared exactly, before and after cleanup. Structure is checked by
    properties that hold at any size."""
    b = 1 << 20
    R = 64
    seed = synth.SEED_BASE + 2
    lo_key, hi_key = 1 << 24, (1 << 24) + (1 << 25)  # 1/64 of the domain
    g = pkg.GpuLSM(b, reserve_batches=R)
    o1 = oracle.OracleDict(b)
    for j in range(R):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=1)
        g.update(to_device(k), to_device(v), to_device(d))
        sel = (k >= lo_key) & (k < hi_key)
        o1.apply_batch(k[sel], v[sel], d[sel])
    g.sync()
    assert g.r == R

    def check(tag):
        rng = np.random.default_rng(7)
        q = np.concatenate([o1.items()[0][:20000],
                            rng.integers(lo_key, hi_key, 20000).astype(np.uint32)])
        gv, gf = g.lookup(to_device(q))
        ov, of = o1.lookup(q)
        assert np.array_equal(gf.cpu().numpy(), of), tag
        assert np.array_equal(to_numpy_u32(gv), ov), tag
        w = 8 * synth.D // (R * b)
        k1 = rng.integers(lo_key, hi_key - w, 5000).astype(np.uint32)
        k2 = (k1 + w).astype(np.uint32)
        gc = to_numpy_u32(g.count(to_device(k1), to_device(k2)))
        assert np.array_equal(gc, o1.count(k1, k2)), tag
        off, ks, vs = g.range(to_device(k1), to_device(k2))
        ooff, oks, ovs = o1.range(k1, k2)
        assert np.array_equal(off.cpu().numpy().astype(np.uint64), ooff), tag
        assert np.array_equal(to_numpy_u32(ks), oks) and np.array_equal(to_numpy_u32(vs), ovs)

    def props():
        for i in range(g.r.bit_length()):
            k, _ = g.level(i)
            kk = to_numpy_u32(k)
            if (g.r >> i) & 1:
                assert len(kk) == b << i
                assert np.all((kk[1:] >> 1) >= (kk[:-1] >> 1))
            else:
                assert len(kk) == 0

    props()
    check("before cleanup")
    g.cleanup()
    assert g.r == -(-len_live(g) // b)
    props()
    check("after cleanup")


def len_live(g):
    tot = 0
    for i in range(g.r.bit_length()):
        k, _ = g.level(i)
        kk = to_numpy_u32(k)
        tot += int(np.count_nonzero(kk & 1))
    return tot


def test_successor_predecessor_tombstone_runs_and_many_levels():
    # Long runs of deleted keys (the walk must skip them), placebo tails from
    # partial batches, queries beyond every key, and r = 511 (9 levels: the
    # generic, non-unrolled kernel).
    b = 64
    gpu, o1 = GpuAdapter(b), oracle.OracleDict(b)
    rng = np.random.default_rng(77)
    q = np.concatenate([np.arange(0, 4200, 7, dtype=np.uint32),
                        np.array([0, 1, 4095, 4096, 0x7FFFFFFE, 0x7FFFFFFF, 0x80000000,
                                  0xFFFFFFFF], np.uint32)])
    for j in range(511):
        if j < 40:  # dense inserts of keys 0..2559
            k = np.arange(j * b, (j + 1) * b, dtype=np.uint32)
            d = np.zeros(b, np.uint8)
        elif j < 60:  # delete a contiguous block -> long tombstone stretch
            k = np.arange(1000 + (j - 40) * b, 1000 + (j - 39) * b, dtype=np.uint32)
            d = np.ones(b, np.uint8)
        else:
            n = int(rng.integers(1, b + 1))  # partial batches: placebo padding
            k = rng.integers(0, 4096, n).astype(np.uint32)
            d = (rng.integers(0, 4, n) == 0).astype(np.uint8)
        v = np.arange(j * b, j * b + len(k), dtype=np.uint32)
        gpu.update(k, v, d)
        o1.apply_batch(k, v, d)
        if j in (0, 39, 59, 60, 127, 255, 300, 510):
            assert_order_equal(gpu, o1, q, f"batch {j}")
    assert gpu.r == 511
    gpu.cleanup()
    o1.cleanup()
    assert_order_equal(gpu, o1, q, "after cleanup")
    # everything deleted -> no successor / predecessor anywhere
    gpu2, o2 = GpuAdapter(8), oracle.OracleDict(8)
    k = np.arange(8, dtype=np.uint32)
    for d in (np.zeros(8, np.uint8), np.ones(8, np.uint8)):
        gpu2.update(k, k, d)
        o2.apply_batch(k, k, d)
    assert_order_equal(gpu2, o2, np.arange(12, dtype=np.uint32), "all deleted")
    gk, _, gf = gpu2.successor(np.arange(12, dtype=np.uint32))
    assert not gf.any() and np.all(gk == 0xFFFFFFFF)


@pytest.mark.parametrize("b,n", [(64, 1), (64, 64), (64, 1000), (4096, 4096 * 5 + 17),
                                 (1 << 16, (1 << 16) * 3), (1 << 20, (1 << 20) * 3 + 5)])
def test_bulk_build(b, n):
    # N1: one sort + level views; bit-exact vs S1, queries vs O1,
    # then ordinary batches on top (newer than the bulk epoch) and a cleanup.
    seed = synth.SEED_BASE + 50 + n % 97
    k, v, d = synth.updates(seed, 0, n, delete_frac4=1, alphabet=max(8, n // 2))
    gpu, s1, o1 = GpuAdapter(b), oracle.ShadowLSM(b), oracle.OracleDict(b)
    gpu.lsm.bulk_build(to_device(k), to_device(v), to_device(d))
    s1.bulk_build(k, v, d)
    o1.bulk_build(k, v, d)
    assert gpu.r == s1.r == o1.r == -(-n // b)
    assert_levels_equal(gpu, s1, "bulk")
    q = synth.lookup_queries(seed, 3000, n, alphabet=max(8, n // 2))
    k1, k2 = synth.range_queries(seed, 500, max(n, 1), 8, domain=max(8, n // 2))
    assert_queries_equal(gpu, o1, q, k1, k2, "bulk")
    for j in range(3):
        kk, vv, dd = synth.updates(seed, n + j * b, b, delete_frac4=1, alphabet=max(8, n // 2))
        gpu.update(kk, vv, dd)
        s1.update(kk, vv, dd)
        o1.apply_batch(kk, vv, dd)
        assert_levels_equal(gpu, s1, f"bulk+{j}")
    assert_queries_equal(gpu, o1, q, k1, k2, "bulk+3")
    gpu.cleanup()
    s1.cleanup()
    o1.cleanup()
    assert_levels_equal(gpu, s1, "bulk cleanup")


def test_bulk_build_errors():
    g = pkg.GpuLSM(64)
    k = to_device(np.arange(10, dtype=np.uint32))
    with pytest.raises(pkg.LsmError):
        g.bulk_build(k[:0])
    g.bulk_build(k, k)
    with pytest.raises(pkg.LsmError):  # only into an empty structure
        g.bulk_build(k, k)


@pytest.mark.parametrize("b,nb,r0", [(64, 13, 0), (64, 9, 5), (1000, 7, 3), (4096, 6, 1),
                                     (10_000, 5, 2), (1 << 17, 3, 1)])
def test_update_batches_equals_sequential(b, nb, r0):
    # N1 multi-batch insertion (PAPER.md:860 footnote): bit-exact equal to nb
    # sequential lsm_update calls (S1), the last batch partial.
    seed = synth.SEED_BASE + 60 + b % 89
    gpu, s1, o1 = GpuAdapter(b), oracle.ShadowLSM(b), oracle.OracleDict(b)
    for j in range(r0):
        kk, vv, dd = synth.updates(seed, j * b, b, delete_frac4=1, alphabet=3 * b)
        gpu.update(kk, vv, dd)
        s1.update(kk, vv, dd)
        o1.apply_batch(kk, vv, dd)
    n = nb * b - b // 3
    k, v, d = synth.updates(seed, r0 * b, n, delete_frac4=1, alphabet=3 * b)
    gpu.lsm.update_batches(to_device(k), to_device(v), to_device(d))
    for j in range(nb):
        sl = slice(j * b, min(n, (j + 1) * b))
        s1.update(k[sl], v[sl], d[sl])
        o1.apply_batch(k[sl], v[sl], d[sl])
    assert gpu.r == s1.r == r0 + nb
    assert_levels_equal(gpu, s1, "multi")
    q = synth.lookup_queries(seed, 2000, (r0 + nb) * b, alphabet=3 * b)
    k1, k2 = synth.range_queries(seed, 300, (r0 + nb) * b, 8, domain=3 * b)
    assert_queries_equal(gpu, o1, q, k1, k2, "multi")


class GpuSAAdapter(GpuAdapter):
    def __init__(self, b):
        self.lsm = pkg.GpuLSM(b, sa=True)


def assert_sa_equal(gpu, sa, where=""):
    gk, gv = gpu.level(0)
    ak, av = sa.array()
    assert gpu.r == sa.r, where
    assert np.array_equal(gk, ak), f"{where} SA keys differ at {np.nonzero(gk != ak)[0][:8]}"
    assert np.array_equal(gv, av), f"{where} SA vals differ"
    for i in range(1, 6):
        assert len(gpu.level(i)[0]) == 0


@pytest.mark.parametrize("b", [4, 100, 4096, 1 << 16])
def test_gpu_sa(b):
    # N2: the one-array structure, bit-exact vs the oracle's
    # SA after every batch; queries (one level) vs O1; cleanup; more batches.
    seed = synth.SEED_BASE + 80 + b % 13
    gpu, sa, o1 = GpuSAAdapter(b), oracle.ShadowSA(b), oracle.OracleDict(b)
    nb = 12 if b <= 4096 else 5
    alpha = 3 * b
    for j in range(nb):
        n = b if j % 4 else max(1, b - b // 3)
        k, v, d = synth.updates(seed, j * b, n, delete_frac4=1, alphabet=alpha)
        gpu.update(k, v, d)
        sa.update(k, v, d)
        o1.apply_batch(k, v, d)
        assert_sa_equal(gpu, sa, f"batch {j}")
    q = synth.lookup_queries(seed, 3000, nb * b, alphabet=alpha)
    k1, k2 = synth.range_queries(seed, 500, nb * b, 8, domain=alpha)
    assert_queries_equal(gpu, o1, q, k1, k2, "sa")
    gpu.cleanup()
    sa.cleanup()
    o1.cleanup()
    assert_sa_equal(gpu, sa, "sa cleanup")
    assert_queries_equal(gpu, o1, q, k1, k2, "sa cleanup")
    k, v, d = synth.updates(seed, nb * b, b, delete_frac4=1, alphabet=alpha)
    gpu.update(k, v, d)
    sa.update(k, v, d)
    o1.apply_batch(k, v, d)
    assert_sa_equal(gpu, sa, "sa after cleanup")
    assert_queries_equal(gpu, o1, q, k1, k2, "sa after cleanup")


def test_gpu_sa_bulk_and_multi_batch():
    b = 64
    seed = synth.SEED_BASE + 81
    k, v, d = synth.updates(seed, 0, 1000, delete_frac4=1, alphabet=300)
    gpu, sa, o1 = GpuSAAdapter(b), oracle.ShadowSA(b), oracle.OracleDict(b)
    gpu.lsm.bulk_build(to_device(k), to_device(v), to_device(d))
    sa.bulk_build(k, v, d)
    o1.bulk_build(k, v, d)
    assert_sa_equal(gpu, sa, "sa bulk")
    k2_, v2_, d2_ = synth.updates(seed, 1000, 5 * b - 7, delete_frac4=1, alphabet=300)
    gpu.lsm.update_batches(to_device(k2_), to_device(v2_), to_device(d2_))
    for j in range(5):
        sl = slice(j * b, min(len(k2_), (j + 1) * b))
        sa.update(k2_[sl], v2_[sl], d2_[sl])
        o1.apply_batch(k2_[sl], v2_[sl], d2_[sl])
    assert_sa_equal(gpu, sa, "sa multi")
    q = synth.lookup_queries(seed, 2000, 1400, alphabet=300)
    k1, kk2 = synth.range_queries(seed, 300, 1400, 8, domain=300)
    assert_queries_equal(gpu, o1, q, k1, kk2, "sa multi")


@pytest.mark.slow
def test_config_c2_full():
    # BASELINE configs[1] (C2): b = 2^16, insert-only, R = 64 batches from
    # empty; lookups, counts and ranges at L = 8 at r in {1, 3, 7, 15, 31, 63,
    # 64} (the occupancy patterns of Table II-IV), exact vs O1 on samples of
    # the paper's nq = n protocol.
    b = 1 << 16
    seed = synth.SEED_BASE + 1
    g = GpuAdapter(b)
    o1 = oracle.OracleDict(b)
    check_at = {1, 3, 7, 15, 31, 63, 64}
    for j in range(64):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=0)
        g.update(k, v, d)
        o1.apply_batch(k, v, d)
        r = j + 1
        if r in check_at:
            n = r * b
            q = synth.lookup_queries(seed, 50_000, n)
            k1, k2 = synth.range_queries(seed, 20_000, n, 8)
            assert_queries_equal(g, o1, q, k1, k2, f"C2 r={r}")


@pytest.mark.slow
def test_config_c4_shape_sampled():
    # BASELINE configs[3] (C4) shape: b = 2^20, insert-only, r = 127 (seven
    # occupied levels, n = 127 * 2^20), queries at L in {8, 64, 1024}. O1 is
    # fed the updates of one key sub-range (exact: keys never interact); the
    # answers it can vouch for are compared.
    b = 1 << 20
    R = 127
    seed = synth.SEED_BASE + 3
    lo_key, hi_key = 3 << 25, (3 << 25) + (1 << 25)  # 1/64 of the domain
    g = pkg.GpuLSM(b, reserve_batches=R)
    o1 = oracle.OracleDict(b)
    for j in range(R):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=0)
        g.update(to_device(k), to_device(v), to_device(d))
        sel = (k >= lo_key) & (k < hi_key)
        o1.apply_batch(k[sel], v[sel], d[sel])
    g.sync()
    assert g.r == R
    n = R * b
    rng = np.random.default_rng(11)
    for L in (8, 64, 1024):
        w = max(1, round(L * synth.D / n))
        k1 = rng.integers(lo_key, hi_key - w, 4000).astype(np.uint32)
        k2 = (k1 + w - 1).astype(np.uint32)
        gc = to_numpy_u32(g.count(to_device(k1), to_device(k2)))
        assert np.array_equal(gc, o1.count(k1, k2)), L
        assert abs(gc.mean() - L) < 0.2 * L + 2, (L, gc.mean())  # R15: E[count] = L
        off, ks, vs = g.range(to_device(k1), to_device(k2))
        ooff, oks, ovs = o1.range(k1, k2)
        assert np.array_equal(off.cpu().numpy().astype(np.uint64), ooff), L
        assert np.array_equal(to_numpy_u32(ks), oks) and np.array_equal(to_numpy_u32(vs), ovs), L
    q = np.concatenate([o1.items()[0][::7][:20000],
                        rng.integers(lo_key, hi_key, 20000).astype(np.uint32)])
    gv, gf = g.lookup(to_device(q))
    ov, of = o1.lookup(q)
    assert np.array_equal(gf.cpu().numpy(), of) and np.array_equal(to_numpy_u32(gv), ov)
    for name in ("successor", "predecessor"):
        gk, gvv, gff = getattr(g, name)(to_device(q))
        ok, ovv, off_ = getattr(o1, name)(q)
        sure = off_ == 1  # an answer inside the sub-range is the global answer
        assert np.array_equal(to_numpy_u32(gk)[sure], ok[sure]), name
        assert np.array_equal(to_numpy_u32(gvv)[sure], ovv[sure]), name
        assert np.all(gff.cpu().numpy()[sure] == 1), name


def test_cascade_concentrated_batch():
    # batches whose keys all fall into one narrow key range (400 keys) merged
    # into uniform levels by t = 3 cascades: every merge tile (and every
    # prefix chunk of a partitioned merge) straddling that range is dominated
    # by one run -- bit-exact vs S1 regardless.
    b = 8192
    gpu, s1, o1 = GpuAdapter(b), oracle.ShadowLSM(b), oracle.OracleDict(b)
    seed = synth.SEED_BASE + 95
    for j in range(15):
        if j in (7, 14):  # t = 3 cascades with a concentrated batch
            rng = np.random.default_rng(j)
            k = rng.integers(1_000_000, 1_000_400, b).astype(np.uint32)
            v = np.arange(j * b, (j + 1) * b, dtype=np.uint32)
            d = (rng.integers(0, 4, b) == 0).astype(np.uint8)
        else:
            k, v, d = synth.updates(seed, j * b, b, delete_frac4=1, alphabet=4_000_000)
        gpu.update(k, v, d)
        s1.update(k, v, d)
        o1.apply_batch(k, v, d)
        assert_levels_equal(gpu, s1, f"batch {j}")
    q = np.concatenate([np.arange(999_990, 1_000_410, dtype=np.uint32),
                        synth.lookup_queries(seed, 2000, 15 * b, alphabet=4_000_000)])
    k1 = np.array([999_000, 1_000_100, 0], np.uint32)
    k2 = np.array([1_000_500, 1_000_200, 4_000_000], np.uint32)
    assert_queries_equal(gpu, o1, q, k1, k2, "skewed")


def test_concentrated_batches_and_cleanup():
    # one-wave batches (b = 32768) whose keys all lie in 400 consecutive keys:
    # oversized sort buckets and merge tiles dominated by one run, then a
    # cleanup merging several such levels -- bit-exact vs S1 regardless.
    b = 32768
    gpu, s1, o1 = GpuAdapter(b), oracle.ShadowLSM(b), oracle.OracleDict(b)
    seed = synth.SEED_BASE + 96
    for j in range(15):
        if j in (3, 7, 14):
            rng = np.random.default_rng(j)
            k = rng.integers(1_000_000, 1_000_400, b).astype(np.uint32)
            v = np.arange(j * b, (j + 1) * b, dtype=np.uint32)
            d = (rng.integers(0, 4, b) == 0).astype(np.uint8)
        else:
            k, v, d = synth.updates(seed, j * b, b, delete_frac4=1, alphabet=4_000_000)
        gpu.update(k, v, d)
        s1.update(k, v, d)
        o1.apply_batch(k, v, d)
        assert_levels_equal(gpu, s1, f"batch {j}")
    q = np.concatenate([np.arange(999_990, 1_000_410, dtype=np.uint32),
                        synth.lookup_queries(seed, 2000, 15 * b, alphabet=4_000_000)])
    k1 = np.array([999_000, 1_000_100, 0], np.uint32)
    k2 = np.array([1_000_500, 1_000_200, 4_000_000], np.uint32)
    assert_queries_equal(gpu, o1, q, k1, k2, "concentrated")
    gpu.cleanup()
    s1.cleanup()
    o1.cleanup()
    assert_levels_equal(gpu, s1, "concentrated cleanup")
    assert_queries_equal(gpu, o1, q, k1, k2, "concentrated cleanup")


def test_nine_levels_r257():
    # r up to 257 with b = 32768: cascades up to t = 8 (nine levels merged at
    # r = 255) and the >8-level query kernels at r = 255
    b = 32768
    gpu, s1, o1 = GpuAdapter(b), oracle.ShadowLSM(b), oracle.OracleDict(b)
    seed = synth.SEED_BASE + 97
    for j in range(257):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=1)
        gpu.update(k, v, d)
        s1.update(k, v, d)
        o1.apply_batch(k, v, d)
        if j + 1 in (3, 8, 127, 255, 256, 257):
            assert_levels_equal(gpu, s1, f"r={j + 1}")
    q = synth.lookup_queries(seed, 20_000, 257 * b)
    k1, k2 = synth.range_queries(seed, 5000, 257 * b, 8)
    assert_queries_equal(gpu, o1, q, k1, k2, "r=257")


def test_unaligned_views():
    # b = 40003 (odd): staged batches, cleanup views and bulk-build views start
    # at element offsets that are not 16-byte aligned; the merges' staging
    # copies read aligned supersets around them
    b = 40003
    _run_schedule(b, 11, synth.SEED_BASE + 98, frac4=1, alphabet=200_000, nlook=3000,
                  nrange=500, cleanup_every=5)
    gpu, s1 = GpuAdapter(b), oracle.ShadowLSM(b)
    k, v, d = synth.updates(synth.SEED_BASE + 99, 0, 5 * b + 7, delete_frac4=1)
    gpu.lsm.bulk_build(to_device(k), to_device(v), to_device(d))
    s1.bulk_build(k, v, d)
    for j in range(3):
        kk, vv, dd = synth.updates(synth.SEED_BASE + 99, 6 * b + j * b, b, delete_frac4=1)
        gpu.update(kk, vv, dd)
        s1.update(kk, vv, dd)
        assert_levels_equal(gpu, s1, f"bulk+{j}")
    k2_, v2_, d2_ = synth.updates(synth.SEED_BASE + 99, 20 * b, 3 * b - 11, delete_frac4=1)
    gpu.lsm.update_batches(to_device(k2_), to_device(v2_), to_device(d2_))
    for j in range(3):
        sl = slice(j * b, min(len(k2_), (j + 1) * b))
        s1.update(k2_[sl], v2_[sl], d2_[sl])
    assert_levels_equal(gpu, s1, "multi on views")


def test_torch_caching_allocator_hook():
    # lsm_create_with_allocator: levels and scratch come from
    # torch's caching allocator; results bit-exact as with the library's pool
    b = 4096
    before = torch.cuda.memory_allocated()
    g = pkg.GpuLSM(b, allocator="torch")
    s1, o1 = oracle.ShadowLSM(b), oracle.OracleDict(b)
    seed = synth.SEED_BASE + 55
    for j in range(11):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=1, alphabet=30_000)
        g.update(to_device(k), to_device(v), to_device(d))
        s1.update(k, v, d)
        o1.apply_batch(k, v, d)
    assert torch.cuda.memory_allocated() > before  # the handle's memory is torch's
    for i in range(s1.num_levels()):
        gk, gv = g.level(i)
        sk, sv = s1.level(i)
        assert np.array_equal(to_numpy_u32(gk), sk) and np.array_equal(to_numpy_u32(gv), sv)
    q = synth.lookup_queries(seed, 5000, 11 * b, alphabet=30_000)
    gv_, gf_ = g.lookup(to_device(q))
    ov, of = o1.lookup(q)
    assert np.array_equal(gf_.cpu().numpy(), of) and np.array_equal(to_numpy_u32(gv_), ov)
    g.cleanup()
    o1.cleanup()
    gv_, gf_ = g.lookup(to_device(q))
    assert np.array_equal(gf_.cpu().numpy(), of) and np.array_equal(to_numpy_u32(gv_), ov)
    g.close()


@pytest.mark.slow
def test_two_level_sort_top_digit_overflow():
    # b = 2^21 + 5 takes the two-level MSD sort; 30 % of the keys share top
    # digit 7 (k >> 23 == 7), far over its region: that digit is regathered
    # from the raw batch and sorted by the chunked LSD -- bit-exact vs S1
    b = (1 << 21) + 5

    def keyfn(h0, h5):
        uni = synth.mulhi(h0, synth.D)
        hot = np.uint64(7 << 23) + (h0 & np.uint64((1 << 23) - 1))
        return np.where(h5 % np.uint64(10) < np.uint64(3), hot, uni)
    _run_custom_keys(b, 3, 4242, keyfn)


@pytest.mark.slow
def test_two_level_sort_sub_bucket_overflow():
    # b = 2^22 (w = 2 sub-digit bits): 6000 keys fall into sub-bucket (top
    # digit 9, sub-digit 1) and no other key has top digit 9, so only that
    # sub-bucket exceeds its 5632-record region
    b = 1 << 22

    def keyfn(h0, h5):
        uni = synth.mulhi(h0, synth.D)
        uni = np.where((uni >> np.uint64(23)) == np.uint64(9), uni ^ np.uint64(1 << 27), uni)
        hot = np.uint64((9 << 23) | (1 << 21)) + (h0 & np.uint64((1 << 21) - 1))
        return np.where(h5 % np.uint64(b) < np.uint64(6000), hot, uni)
    _run_custom_keys(b, 2, 4343, keyfn)


@pytest.mark.slow
def test_two_level_sort_duplicates():
    # duplicate-heavy keys at b = 2^21 + 77: position tie-breaks with 27-bit
    # positions in the two-level rank pass (first insert wins, R4)
    _run_schedule((1 << 21) + 77, 3, 4444, frac4=1, alphabet=500_000, nlook=20_000, nrange=1000)


@pytest.mark.slow
def test_multi_wave_lsd_after_skew():
    # b = 2^21 + 4097 with keys < 3000: the first batch's single top digit
    # overflows the two-level sort (one CTA regathers and LSD-sorts it), which
    # moves the handle to the multi-wave onesweep LSD (tile counter, group
    # look-back) for the later batches -- all bit-exact vs S1
    _run_schedule((1 << 21) + 4097, 3, 4545, frac4=1, alphabet=3000, nlook=3000, nrange=300)
