"""Pins for the CPU oracle (O1 map, S1 structural LSM) -- CPU only.

Each test pins the oracle to something other than itself: the paper's and
SPEC's worked examples (tests/golden/*.lsm, each with its citation), closed
forms of the merge work, structural invariants
(PAPER.md:377-382, 417-429), and brute force O0 (oracle/brute.py) on
exhaustive tiny schedules.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from tests import lsm_script


class OracleAdapter:
    """Structure from S1; every query answered by S1 (paper pipeline) AND O1
    (definition), asserted equal."""

    def __init__(self, b):
        self.s1 = oracle.ShadowLSM(b)
        self.o1 = oracle.OracleDict(b)

    def update(self, k, v, d):
        self.s1.update(k, v, d)
        self.o1.apply_batch(k, v, d)

    def lookup(self, q):
        a = self.s1.lookup(q)
        b = self.o1.lookup(q)
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0])
        return a

    def count(self, k1, k2):
        a = self.s1.count(k1, k2)
        assert np.array_equal(a, self.o1.count(k1, k2))
        return a

    def range(self, k1, k2):
        a = self.s1.range(k1, k2)
        b = self.o1.range(k1, k2)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        return a

    def cleanup(self):
        self.s1.cleanup()
        self.o1.cleanup()
        assert self.s1.r == self.o1.r

    @property
    def r(self):
        return self.s1.r

    @property
    def merged_records(self):
        return self.s1.merged_records

    def level(self, i):
        return self.s1.level(i)

    def num_levels(self):
        return self.s1.num_levels()


@pytest.mark.parametrize("path", lsm_script.golden_files(), ids=lambda p: p.split("/")[-1])
def test_golden_scripts(path):
    lsm_script.run(path, OracleAdapter)


def test_text_dump_matches_script_dump():
    s = oracle.ShadowLSM(4)
    s.update(np.array([3, 7], np.uint32), np.array([1, 2], np.uint32), np.array([0, 1], np.uint8))
    assert oracle.dump_text(s) == "lsm b=4 r=1\nlevel 0: 3:R:1 7:T:0 " \
        "2147483647:T:0 2147483647:T:0"


def test_bounds_spec_examples():
    # keys [2,4,4,9] (original keys; packed = k<<1|1)
    packed = [(k << 1) | 1 for k in (2, 4, 4, 9)]
    assert oracle.lower_bound(packed, 4) == 1
    assert oracle.lower_bound(packed, 10) == 4
    assert oracle.upper_bound(packed, 4) == 3
    assert oracle.upper_bound(packed, 1) == 0
    # status bit ignored: a tombstone 4 is still "equal" to 4
    packed2 = [(2 << 1) | 1, (4 << 1), (4 << 1) | 1, (9 << 1)]
    assert oracle.lower_bound(packed2, 4) == 1 and oracle.upper_bound(packed2, 4) == 3
    # query keys >= 2^31 compared unshifted (R8): never equal to a stored key
    assert oracle.lower_bound(packed, 0xFFFFFFFF) == 4


def test_bounds_vs_linear_scan_exhaustive():
    # bounds match linear scans on sorted inputs (brute force)
    rng = np.random.default_rng(1)
    for n in range(0, 20):
        for _ in range(20):
            ks = np.sort(rng.integers(0, 6, n)) if n else np.zeros(0, np.int64)
            st = rng.integers(0, 2, n)
            packed = [(int(k) << 1) | int(s) for k, s in zip(ks, st)]
            for q in range(-0, 8):
                lb = next((i for i, k in enumerate(ks) if k >= q), n)
                ub = next((i for i, k in enumerate(ks) if k > q), n)
                assert oracle.lower_bound(packed, q) == lb
                assert oracle.upper_bound(packed, q) == ub


def _ffz(r):
    t = 0
    while (r >> t) & 1:
        t += 1
    return t


@pytest.mark.parametrize("b", [1, 3, 8])
def test_merge_work_closed_form_and_occupancy(b):
    # T_ins(r) = T_sort + (2^ffz(r)-1) T_merge  =>  each insert
    # at r writes exactly 2b(2^ffz(r)-1) merged records.
    # occupied levels are the set bits of r.
    s = oracle.ShadowLSM(b)
    total = 0
    for r in range(0, 70):
        before = s.merged_records
        k, v, d = synth.updates(7, r * b, b, delete_frac4=1)
        s.update(k, v, d)
        delta = s.merged_records - before
        assert delta == 2 * b * (2 ** _ffz(r) - 1)
        total += delta
        R = r + 1
        occ = [i for i in range(s.num_levels()) if len(s.level(i)[0]) > 0]
        assert occ == [i for i in range(R.bit_length()) if (R >> i) & 1]
        for i in occ:
            assert len(s.level(i)[0]) == b << i
        # amortized bound
        assert s.merged_records <= 2 * b * R * math.ceil(math.log2(R + 1))
        # exact closed form at R = 2^m (derived): b * R * log2 R
        if R & (R - 1) == 0:
            assert s.merged_records == b * R * int(math.log2(R))


def test_building_invariants_random():
    # (1) each level sorted by key; (2) within a segment,
    # newest first; (3) within one batch, tombstones before regulars (R3).
    b = 16
    s = oracle.ShadowLSM(b)
    for j in range(40):
        k, v, d = synth.updates(11, j * b, b, delete_frac4=2, alphabet=24)
        s.update(k, v, d)
        for i in range(s.num_levels()):
            keys, vals, tags = s.level(i, with_tags=True)
            if len(keys) == 0:
                continue
            orig = keys >> 1
            assert np.all(orig[1:] >= orig[:-1])
            same = orig[1:] == orig[:-1]
            assert np.all(tags[1:][same] <= tags[:-1][same])          # (2)
            same_batch = same & (tags[1:] == tags[:-1])
            assert np.all((keys[1:] & 1)[same_batch] >= (keys[:-1] & 1)[same_batch])  # (3)
            assert np.all(vals[(keys & 1) == 0] == 0)  # R6


def _sorted_by_definition(recs):
    # stable sort by packed key: explicit (key, input index)
    return [r for _, _, r in sorted((r[0], i, r) for i, r in enumerate(recs))]


def test_sort_and_merge_exhaustive_tiny():
    # merge == stable sort keyed on (original key, source
    # newer=0/older=1, index), exhaustive over a 3-key alphabet with ops {I,D},
    # b = 2 (combined merge size 4) plus all single batches of b = 3.
    ops = [(k, d) for k in range(3) for d in (0, 1)]
    for b, nb in ((3, 1), (2, 2)):
        for combo in itertools.product(ops, repeat=b * nb):
            s = oracle.ShadowLSM(b)
            sorted_batches = []
            for j in range(nb):
                part = combo[j * b:(j + 1) * b]
                keys = np.array([k for k, _ in part], np.uint32)
                dels = np.array([d for _, d in part], np.uint8)
                vals = np.arange(j * b + 1, (j + 1) * b + 1, dtype=np.uint32)
                s.update(keys, vals, dels)
                recs = [((int(k) << 1) | (0 if d else 1), 0 if d else int(v))
                        for k, d, v in zip(keys, dels, vals)]
                sorted_batches.append(_sorted_by_definition(recs))
            if nb == 1:
                exp = sorted_batches[0]
                lvl = 0
            else:
                newer, older = sorted_batches[1], sorted_batches[0]
                tagged = [(r[0] >> 1, 0, i, r) for i, r in enumerate(newer)] + \
                         [(r[0] >> 1, 1, i, r) for i, r in enumerate(older)]
                exp = [t[3] for t in sorted(tagged)]
                lvl = 1
            k, v = s.level(lvl)
            assert list(zip(k.tolist(), v.tolist())) == exp, combo


def _random_schedule_check(b, nbatch, alphabet, seed, frac4, brute=False):
    s = oracle.ShadowLSM(b)
    o = oracle.OracleDict(b)
    o0 = oracle.BruteDict() if brute else None
    dom = alphabet + 2
    for j in range(nbatch):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=frac4, alphabet=alphabet)
        s.update(k, v, d)
        o.apply_batch(k, v, d)
        if o0 is not None:
            o0.apply_batch(k, v, d)
        q = np.arange(dom, dtype=np.uint32)
        sv, sf = s.lookup(q)
        ov, of = o.lookup(q)
        assert np.array_equal(sf, of) and np.array_equal(sv[sf == 1], ov[of == 1])
        k1 = synth.uniform_u32(seed + j, 6, 40) % np.uint32(dom)
        k2 = synth.uniform_u32(seed + j, 7, 40) % np.uint32(dom)
        assert np.array_equal(s.count(k1, k2), o.count(k1, k2))
        for x, y in zip(s.range(k1, k2), o.range(k1, k2)):
            assert np.array_equal(x, y)
        if o0 is not None:
            for qq in range(dom):
                bv = o0.lookup(qq)
                assert (bv is None) == (of[qq] == 0)
                if bv is not None:
                    assert bv == ov[qq]
            for a1, a2 in zip(k1[:10], k2[:10]):
                assert o0.count(a1, a2) == int(o.count([a1], [a2])[0])
                off, ks, vs = o.range([a1], [a2])
                assert o0.range(a1, a2) == list(zip(ks.tolist(), vs.tolist()))
    return s, o


def test_o1_vs_brute_exhaustive_tiny():
    # Whole-pipeline brute force: b = 2, 3-key alphabet,
    # ops {I, D}, all schedules of 2 batches; O0 vs O1 vs S1.
    ops = [(k, d) for k in range(3) for d in (0, 1)]
    b = 2
    for combo in itertools.product(ops, repeat=2 * b):
        s = oracle.ShadowLSM(b)
        o = oracle.OracleDict(b)
        o0 = oracle.BruteDict()
        for j in range(2):
            part = combo[j * b:(j + 1) * b]
            keys = np.array([k for k, _ in part], np.uint32)
            dels = np.array([d for _, d in part], np.uint8)
            vals = np.arange(j * b + 1, (j + 1) * b + 1, dtype=np.uint32)
            for m in (s.update, o.apply_batch, o0.apply_batch):
                m(keys, vals, dels)
            q = np.arange(4, dtype=np.uint32)
            sv, sf = s.lookup(q)
            ov, of = o.lookup(q)
            for qq in range(4):
                bv = o0.lookup(qq)
                assert (bv is None) == (of[qq] == 0) == (sf[qq] == 0), combo
                if bv is not None:
                    assert bv == ov[qq] == sv[qq], combo
            assert o0.count(0, 3) == int(o.count([0], [3])[0]) == int(s.count([0], [3])[0])
        s.cleanup()
        sv2, sf2 = s.lookup(np.arange(4, dtype=np.uint32))
        assert np.array_equal(sf2, of) and np.array_equal(sv2[sf2 == 1], ov[of == 1])


@pytest.mark.parametrize("b,nbatch,alphabet", [(4, 2, 3), (2, 3, 3), (1, 6, 3), (3, 3, 2)])
def test_oracle_exhaustive_schedules(b, nbatch, alphabet):
    # EVERY schedule of nbatch batches of b updates over
    # `alphabet` keys x {insert, delete} ((2A)^(b*nbatch): 6^8 = 1,679,616 for
    # b = 4 and two batches) through three implementations sharing no logic --
    # O0, a literal history scan of the batch rules, O1 and
    # S1 -- compared on lookups after every batch, count / range of every
    # interval and successor / predecessor after the last, and lookups after
    # cleanup (oracle/exhaustive.cpp). A mutant O0 (last insert wins instead of
    # the first, R4) fails at schedule 0.
    n = oracle.exhaustive(b, nbatch, alphabet)
    assert n == (2 * alphabet) ** (b * nbatch)


@pytest.mark.parametrize("seed", range(6))
def test_random_schedules_with_brute(seed):
    _random_schedule_check(b=4, nbatch=12, alphabet=10, seed=seed, frac4=2, brute=True)


@pytest.mark.parametrize("seed", range(8))
def test_random_schedules_s1_vs_o1(seed):
    # SPEC.md:499 acceptance 1 (scaled): duplicate-heavy alphabets, mixed
    s, o = _random_schedule_check(b=64, nbatch=33, alphabet=300, seed=100 + seed, frac4=1)
    # cleanup transparency + idempotence
    q = np.arange(302, dtype=np.uint32)
    before = s.lookup(q)
    k1 = np.array([0, 5, 100], np.uint32)
    k2 = np.array([301, 50, 99], np.uint32)
    rb = s.range(k1, k2)
    s.cleanup()
    o.cleanup()
    after = s.lookup(q)
    assert np.array_equal(before[1], after[1]) and np.array_equal(before[0], after[0])
    for x, y in zip(rb, s.range(k1, k2)):
        assert np.array_equal(x, y)
    assert s.r == o.r == -(-len(o) // 64)
    imgs = [s.level(i) for i in range(s.num_levels())]
    s.cleanup()
    for i, (k, v) in enumerate(imgs):
        k2_, v2_ = s.level(i)
        assert np.array_equal(k, k2_) and np.array_equal(v, v2_)
    # only placebo tombstones remain; no duplicate original keys
    allk = np.concatenate([s.level(i)[0] for i in range(s.num_levels())])
    tomb = allk[(allk & 1) == 0]
    assert np.all(tomb == 0xFFFFFFFE)
    live = allk[(allk & 1) == 1] >> 1
    assert len(np.unique(live)) == len(live) == len(o)


def test_cleanup_image_derivable_from_o1():
    # post-cleanup image = sorted live pairs of O1 encoded
    # (k<<1)|1, then r'b-|S| placebos, sliced into the set bits of r' ascending.
    b = 8
    s, o = _random_schedule_check(b=b, nbatch=21, alphabet=60, seed=5, frac4=2)
    s.cleanup()
    o.cleanup()
    k, v = o.items()
    img_k = np.concatenate([(k.astype(np.uint64) << 1 | 1).astype(np.uint32),
                            np.full(o.r * b - len(k), 0xFFFFFFFE, np.uint32)])
    img_v = np.concatenate([v, np.zeros(o.r * b - len(k), np.uint32)])
    off = 0
    for i in range(64):
        if (o.r >> i) & 1:
            sk, sv = s.level(i)
            n = b << i
            assert np.array_equal(sk, img_k[off:off + n]) and np.array_equal(sv, img_v[off:off + n])
            off += n
    assert off == len(img_k)


def test_count_candidates_scale_with_L():
    # SPEC.md:506 (acceptance 8): mean candidates for L=1024 is 128x L=8 (±20%)
    b = 1 << 12
    s = oracle.ShadowLSM(b)
    for j in range(16):
        k, v, d = synth.updates(3, j * b, b, delete_frac4=0)
        s.update(k, v, d)
    n = 16 * b
    cands = []
    for L in (8, 1024):
        k1, k2 = synth.range_queries(3, 400, n, L)
        _, c = s.count(k1, k2, return_candidates=True)
        cands.append(c / 400)
    assert 0.8 * 128 <= cands[1] / cands[0] <= 1.2 * 128


def test_out_of_domain_key_dropped_with_flag():
    # R5: keys >= 2^31-1 become placebos (S1) / are dropped (O1)
    s = oracle.ShadowLSM(4)
    o = oracle.OracleDict(4)
    k = np.array([5, 0x7FFFFFFF, 0xFFFFFFFF, 6], np.uint32)
    v = np.array([1, 2, 3, 4], np.uint32)
    d = np.zeros(4, np.uint8)
    s.update(k, v, d)
    o.apply_batch(k, v, d)
    assert s.domain_error
    assert len(o) == 2
    kk, vv = s.level(0)
    assert kk.tolist() == [11, 13, 0xFFFFFFFE, 0xFFFFFFFE]


def _succ_pred_brute_check(o, o0, qs):
    ks, vs, fs = o.successor(qs)
    kp, vp, fp = o.predecessor(qs)
    for i, qq in enumerate(qs.tolist()):
        bs, bp = o0.successor(qq), o0.predecessor(qq)
        assert (bs is None) == (fs[i] == 0), (qq, bs)
        assert (bp is None) == (fp[i] == 0), (qq, bp)
        if bs is None:
            assert ks[i] == vs[i] == 0xFFFFFFFF
        else:
            assert (int(ks[i]), int(vs[i])) == bs
        if bp is None:
            assert kp[i] == vp[i] == 0xFFFFFFFF
        else:
            assert (int(kp[i]), int(vp[i])) == bp


def test_successor_predecessor_vs_brute_exhaustive_tiny():
    # N3 (PAPER.md:113 footnote, reading R23) against O0's history scan:
    # b = 2, 3-key alphabet, all 2-batch schedules, every query key 0..3 plus
    # the domain edges.
    ops = [(k, d) for k in range(3) for d in (0, 1)]
    b = 2
    qs = np.array([0, 1, 2, 3, 0x7FFFFFFE, 0x7FFFFFFF, 0xFFFFFFFF], np.uint32)
    for combo in itertools.product(ops, repeat=2 * b):
        o = oracle.OracleDict(b)
        o0 = oracle.BruteDict()
        for j in range(2):
            part = combo[j * b:(j + 1) * b]
            keys = np.array([k for k, _ in part], np.uint32)
            dels = np.array([d for _, d in part], np.uint8)
            vals = np.arange(j * b + 1, (j + 1) * b + 1, dtype=np.uint32)
            o.apply_batch(keys, vals, dels)
            o0.apply_batch(keys, vals, dels)
            _succ_pred_brute_check(o, o0, qs)


@pytest.mark.parametrize("seed", range(4))
def test_successor_predecessor_vs_brute_random(seed):
    rng = np.random.default_rng(900 + seed)
    o = oracle.OracleDict(4)
    o0 = oracle.BruteDict()
    for j in range(10):
        keys = rng.integers(0, 12, 4).astype(np.uint32)
        dels = (rng.integers(0, 3, 4) == 0).astype(np.uint8)
        vals = np.arange(j * 4, j * 4 + 4, dtype=np.uint32)
        o.apply_batch(keys, vals, dels)
        o0.apply_batch(keys, vals, dels)
        _succ_pred_brute_check(o, o0, np.arange(14, dtype=np.uint32))


def test_successor_predecessor_count_invariants():
    # Properties fixed by the definitions, checked through count (itself
    # pinned to O0): succ(q) = s  =>  count(q, s-1) == 0 and count(s, s) == 1;
    # no successor  =>  count(q, MAX) == 0; mirror for pred. lookup(q) found
    # <=> succ(q) == q == pred(q).
    b = 256
    seed = synth.SEED_BASE + 41
    o = oracle.OracleDict(b)
    for j in range(9):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=2, alphabet=2000)
        o.apply_batch(k, v, d)
    qs = np.concatenate([np.arange(0, 2100, dtype=np.uint32),
                         np.array([0x7FFFFFFE, 0x7FFFFFFF, 0xFFFFFFFF], np.uint32)])
    ks, vs, fs = o.successor(qs)
    kp, vp, fp = o.predecessor(qs)
    lv, lf = o.lookup(qs)
    mx = np.full(len(qs), 0x7FFFFFFE, np.uint32)
    zero = np.zeros(len(qs), np.uint32)
    for i, qq in enumerate(qs.tolist()):
        if fs[i]:
            assert ks[i] >= qq
            if ks[i] > qq:
                assert o.count([qq], [ks[i] - 1])[0] == 0
            assert o.count([ks[i]], [ks[i]])[0] == 1
            assert vs[i] == o.lookup([ks[i]])[0][0]
        else:
            assert o.count([min(qq, 0x7FFFFFFF)], [mx[i]])[0] == 0
        if fp[i]:
            assert kp[i] <= qq
            if kp[i] < qq:
                assert o.count([kp[i] + 1], [min(qq, 0xFFFFFFFE)])[0] == 0
            assert o.count([kp[i]], [kp[i]])[0] == 1
        else:
            assert o.count([zero[i]], [qq])[0] == 0
        assert bool(lf[i]) == (bool(fs[i]) and ks[i] == qq) == (bool(fp[i]) and kp[i] == qq)


def test_bulk_build_single_batch_equals_update():
    # k = 1: a bulk build of n <= b elements is one batch inserted into the
    # empty structure, i.e. exactly s1_update's level 0 (pinned by the paper's
    # worked examples above).
    rng = np.random.default_rng(5)
    for n in (1, 7, 64):
        keys = rng.integers(0, 40, n).astype(np.uint32)
        vals = np.arange(n, dtype=np.uint32) + 1
        dels = (rng.integers(0, 4, n) == 0).astype(np.uint8)
        a, c = oracle.ShadowLSM(64), oracle.ShadowLSM(64)
        a.bulk_build(keys, vals, dels)
        c.update(keys, vals, dels)
        assert a.r == c.r == 1
        assert all(np.array_equal(x, y) for x, y in zip(a.level(0), c.level(0)))


def test_bulk_build_image_from_sorted_unique_keys():
    # Unique keys, inserts only: the structure is the sorted pairs encoded
    # (k << 1) | 1, then placebos up to k*b, cut into the set bits of k in
    # ascending order ("segment this array"). Built here with
    # numpy alone.
    b = 16
    rng = np.random.default_rng(11)
    for n in (16, 17, 100, 16 * 7, 16 * 13 - 3):
        keys = rng.choice(1 << 20, n, replace=False).astype(np.uint32)
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        s = oracle.ShadowLSM(b)
        s.bulk_build(keys, vals)
        k = -(-n // b)
        order = np.argsort(keys, kind="stable")
        img_k = np.concatenate([(keys[order] << 1) | 1, np.full(k * b - n, 0xFFFFFFFE, np.uint32)])
        img_v = np.concatenate([vals[order], np.zeros(k * b - n, np.uint32)])
        assert s.r == k
        off = 0
        for i in range(k.bit_length()):
            lk, lv = s.level(i)
            if not (k >> i) & 1:
                assert len(lk) == 0
                continue
            assert np.array_equal(lk, img_k[off:off + (b << i)])
            assert np.array_equal(lv, img_v[off:off + (b << i)])
            off += b << i


@pytest.mark.parametrize("seed", range(3))
def test_bulk_build_queries_vs_brute(seed):
    # Duplicates and deletes inside the bulk input: it is ONE batch (R24), so
    # O0 applies it as one batch; S1 queries and O1 must agree with O0.
    rng = np.random.default_rng(300 + seed)
    b, n = 8, 45
    keys = rng.integers(0, 20, n).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32) + 100
    dels = (rng.integers(0, 4, n) == 0).astype(np.uint8)
    s, o, o0 = oracle.ShadowLSM(b), oracle.OracleDict(b), oracle.BruteDict()
    s.bulk_build(keys, vals, dels)
    o.bulk_build(keys, vals, dels)
    o0.apply_batch(keys, vals, dels)
    assert s.r == o.r == 6
    q = np.arange(22, dtype=np.uint32)
    sv, sf = s.lookup(q)
    ov, of = o.lookup(q)
    for i in range(22):
        bv = o0.lookup(i)
        assert (bv is None) == (sf[i] == 0) == (of[i] == 0)
        if bv is not None:
            assert bv == sv[i] == ov[i]
    for a1, a2 in ((0, 21), (3, 9), (10, 10), (15, 2)):
        assert o0.count(a1, a2) == int(s.count([a1], [a2])[0]) == int(o.count([a1], [a2])[0])
    # later batches are newer than the whole bulk epoch
    k2 = np.array([1, 2, 3], np.uint32)
    v2 = np.array([7, 8, 9], np.uint32)
    d2 = np.array([0, 1, 0], np.uint8)
    s.update(k2, v2, d2)
    o.apply_batch(k2, v2, d2)
    o0.apply_batch(k2, v2, d2)
    sv, sf = s.lookup(q)
    for i in range(22):
        bv = o0.lookup(i)
        assert (bv is None) == (sf[i] == 0)
        if bv is not None:
            assert bv == sv[i]


def _s1_merged_image(s):
    """All S1 levels concatenated newest (lowest index) first, stable-sorted on
    the original key with numpy: the record order both structures must share."""
    ks, vs = [], []
    for i in range(s.num_levels()):
        k, v = s.level(i)
        ks.append(k)
        vs.append(v)
    k = np.concatenate(ks) if ks else np.zeros(0, np.uint32)
    v = np.concatenate(vs) if vs else np.zeros(0, np.uint32)
    o = np.argsort(k >> 1, kind="stable")
    return k[o], v[o]


@pytest.mark.parametrize("seed", range(4))
def test_sa_array_equals_merged_lsm_levels(seed):
    # N2: the SA keeps every record in one array, newest
    # first within a key; the LSM's levels hold the same records split by
    # recency, so their newest-first stable merge (done here by numpy) must be
    # the SA array, bit for bit, after every batch and after cleanup.
    b = 16
    seed = synth.SEED_BASE + 70 + seed
    sa, s1 = oracle.ShadowSA(b), oracle.ShadowLSM(b)
    for j in range(23):
        n = b if j % 5 else b - 5  # partial batches too
        k, v, d = synth.updates(seed, j * b, n, delete_frac4=1, alphabet=60)
        sa.update(k, v, d)
        s1.update(k, v, d)
        ak, av = sa.array()
        mk, mv = _s1_merged_image(s1)
        assert sa.r == s1.r == j + 1 and len(ak) == (j + 1) * b
        assert np.array_equal(ak, mk) and np.array_equal(av, mv)
    sa.cleanup()
    s1.cleanup()
    ak, av = sa.array()
    ck = np.concatenate([s1.level(i)[0] for i in range(s1.num_levels())])
    cv = np.concatenate([s1.level(i)[1] for i in range(s1.num_levels())])
    assert sa.r == s1.r and np.array_equal(ak, ck) and np.array_equal(av, cv)


def test_sa_merge_work_closed_form():
    # SA merge work after r batches = b(r-1)(r+2)/2 records.
    for b in (4, 16):
        sa = oracle.ShadowSA(b)
        for r in range(1, 25):
            k, v, d = synth.updates(synth.SEED_BASE + 71, r * b, b, delete_frac4=0)
            sa.update(k, v, d)
            assert sa.merged_records == b * (r - 1) * (r + 2) // 2


def test_sa_bulk_build_equals_lsm_bulk_image():
    # bulk build of the SA = the LSM bulk image read level by level in
    # ascending order (both are one sort of the padded k*b records, R24)
    b = 8
    k, v, d = synth.updates(synth.SEED_BASE + 72, 0, 45, delete_frac4=1, alphabet=30)
    sa, s1 = oracle.ShadowSA(b), oracle.ShadowLSM(b)
    sa.bulk_build(k, v, d)
    s1.bulk_build(k, v, d)
    ck = np.concatenate([s1.level(i)[0] for i in range(s1.num_levels())])
    cv = np.concatenate([s1.level(i)[1] for i in range(s1.num_levels())])
    ak, av = sa.array()
    assert sa.r == s1.r == 6 and np.array_equal(ak, ck) and np.array_equal(av, cv)


def test_sharded_oracle_equals_o1():
    # the T-thread timing oracle must be O1 exactly
    b = 512
    seed = synth.SEED_BASE + 90
    o, m = oracle.OracleDict(b), oracle.ShardedOracleDict(b, 4)
    for j in range(12):
        k, v, d = synth.updates(seed, j * b, b, delete_frac4=1, alphabet=3000)
        o.apply_batch(k, v, d)
        m.apply_batch(k, v, d)
    q = np.concatenate([np.arange(3100, dtype=np.uint32), np.array([0x7FFFFFFF, 0xFFFFFFFF], np.uint32)])
    assert len(o) == len(m)
    a, b_ = o.lookup(q), m.lookup(q)
    assert np.array_equal(a[0], b_[0]) and np.array_equal(a[1], b_[1])
