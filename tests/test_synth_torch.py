"""The torch (device) copy of the input generator is bit-identical to the numpy
one (synth/__init__.py) -- run on CPU tensors here."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")


def u32(t):
    return t.numpy().view(np.uint32)


@pytest.mark.parametrize("start,count,frac", [(0, 5000, 1), (123456789, 4096, 1), (7, 3000, 0),
                                              ((1 << 33) + 5, 2048, 2)])
def test_updates_bit_identical(start, count, frac):
    k, v, d = synth.updates(synth.SEED_BASE + 2, start, count, delete_frac4=frac)
    tk, tv, td = synth.updates_t(synth.SEED_BASE + 2, start, count, delete_frac4=frac,
                                 device="cpu")
    assert np.array_equal(u32(tk), k)
    assert np.array_equal(u32(tv), v)
    assert np.array_equal(td.numpy(), d)


def test_queries_bit_identical():
    seed = synth.SEED_BASE + 3
    q = synth.lookup_queries(seed, 10000, 1 << 26)
    assert np.array_equal(u32(synth.lookup_queries_t(seed, 10000, 1 << 26, device="cpu")), q)
    for L in (1, 8, 1024, 1e9):
        k1, k2 = synth.range_queries(seed, 5000, 1 << 20, L)
        t1, t2 = synth.range_queries_t(seed, 5000, 1 << 20, L, device="cpu")
        assert np.array_equal(u32(t1), k1) and np.array_equal(u32(t2), k2)
