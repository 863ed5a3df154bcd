"""Seeded synthetic workloads for the GPU LSM hot path (shared input generator).

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle. It holds none of the method's arithmetic: no status-bit encoding, no
sorting, no merging, no dictionary semantics. It only draws numbers.

Generator (SURVEY.md §8(d) "Concrete synthetic inputs"):

    h(seed, stream, i) = splitmix64(seed ^ (stream << 56) ^ i)
    mulhi(h, m)        = floor(h * m / 2^64)            (uniform on [0, m))

Streams: 0 raw insert key, 1 op selector, 2 delete target, 3 fresh query key,
4 hit selector, 5 range lower end.

Workload shapes follow the paper's experiments (§5):
  * keys are "randomly generated" -> uniform original keys on
    [0, 2^31-2] (the 31-bit key domain of §4.1, minus the reserved
    placebo key 2^31-1, reading R5);
  * mixed batches 75% insert / 25% delete (BASELINE.json configs[0], [2]);
  * a delete targets the raw key of a uniformly chosen earlier update, so it
    usually hits a resident key;
  * values are the global update index, so any stale/duplicate mistake shows;
  * lookups: "50% hit" mixes keys of earlier updates with fresh keys;
  * count/range queries of expected resident length L (reading R15):
    width w = max(1, round(L*D/n)), k1 uniform in [0, D-w], k2 = k1+w-1.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
D = (1 << 31) - 1          # size of the user key domain [0, 2^31-2]
SEED_BASE = 1707053540     # + config index


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser over uint64 (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def h(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    salt = np.uint64((seed ^ (stream << 56)) & 0xFFFFFFFFFFFFFFFF)
    return splitmix64(idx ^ salt)


def mulhi(hv: np.ndarray, m) -> np.ndarray:
    """floor(hv * m / 2^64) for m < 2^32 (elementwise m allowed)."""
    m = np.asarray(m, dtype=np.uint64)
    lo = hv & np.uint64(0xFFFFFFFF)
    hi = hv >> np.uint64(32)
    with np.errstate(over="ignore"):
        x = lo * m
        return (hi * m + (x >> np.uint64(32))) >> np.uint64(32)


def raw_keys(seed: int, idx: np.ndarray, alphabet: int | None = None) -> np.ndarray:
    k = mulhi(h(seed, 0, idx), D)
    if alphabet is not None:
        k = k % np.uint64(alphabet)
    return k.astype(np.uint32)


def updates(seed: int, start: int, count: int, delete_frac4: int = 1,
            alphabet: int | None = None):
    """Updates with global indices [start, start+count).

    delete_frac4: number of quarters that are deletes (0 = insert-only,
    1 = 25% deletes). Returns (keys u32, vals u32, is_delete u8).
    """
    idx = np.arange(start, start + count, dtype=np.uint64)
    keys = raw_keys(seed, idx, alphabet)
    vals = idx.astype(np.uint32)
    if delete_frac4 <= 0:
        return keys, vals, np.zeros(count, dtype=np.uint8)
    is_del = (h(seed, 1, idx) % np.uint64(4)) < np.uint64(delete_frac4)
    # a delete targets the raw key of a uniformly chosen earlier update u < i
    safe = np.maximum(idx, np.uint64(1))
    u = mulhi(h(seed, 2, idx), safe)
    tgt = raw_keys(seed, u, alphabet)
    tgt = np.where(idx == 0, keys, tgt)
    keys = np.where(is_del, tgt, keys).astype(np.uint32)
    vals = np.where(is_del, np.uint32(0), vals).astype(np.uint32)
    return keys, vals, is_del.astype(np.uint8)


def batches(seed: int, b: int, nbatches: int, delete_frac4: int = 1,
            alphabet: int | None = None):
    """Yield (keys, vals, is_delete) per batch of exactly b updates."""
    for j in range(nbatches):
        yield updates(seed, j * b, b, delete_frac4, alphabet)


def lookup_queries(seed: int, nq: int, n_updates: int,
                   alphabet: int | None = None) -> np.ndarray:
    """Even-indexed: key of a uniform earlier update; odd: fresh uniform key."""
    j = np.arange(nq, dtype=np.uint64)
    u = mulhi(h(seed, 4, j), max(n_updates, 1))
    hit = raw_keys(seed, u, alphabet)
    fresh = mulhi(h(seed, 3, j), D if alphabet is None else alphabet).astype(np.uint32)
    return np.where((j & np.uint64(1)) == 0, hit, fresh).astype(np.uint32)


def range_queries(seed: int, nq: int, n_resident: int, L: float,
                  domain: int = D):
    """(k1, k2) with expected L resident keys inside (reading R15)."""
    w = max(1, int(round(L * domain / max(n_resident, 1))))
    w = min(w, domain)
    j = np.arange(nq, dtype=np.uint64)
    k1 = mulhi(h(seed, 5, j), domain - w + 1).astype(np.uint32)
    k2 = (k1.astype(np.uint64) + np.uint64(w - 1)).astype(np.uint32)
    return k1, k2


def uniform_u32(seed: int, stream: int, count: int) -> np.ndarray:
    """Arbitrary 32-bit words (edge-case query keys incl. >= 2^31-1)."""
    return (h(seed, stream, np.arange(count, dtype=np.uint64)) >> np.uint64(32)).astype(np.uint32)
