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


# ---------------------------------------------------------------------------
# The same generator on a torch device (bit-identical to the numpy one above;
# pinned by tests/test_synth_torch.py): int64 arithmetic wraps like uint64,
# and right shifts are made logical with a mask. Used to create bench inputs
# directly in device memory.
# ---------------------------------------------------------------------------

def _t():
    import torch
    return torch


def _i64(x):
    """A uint64 constant as the int64 with the same bits."""
    x &= 0xFFFFFFFFFFFFFFFF
    return x - (1 << 64) if x >= (1 << 63) else x


def _lsr(x, k):
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64_t(x):
    z = x + _i64(0x9E3779B97F4A7C15)
    z = (z ^ _lsr(z, 30)) * _i64(0xBF58476D1CE4E5B9)
    z = (z ^ _lsr(z, 27)) * _i64(0x94D049BB133111EB)
    return z ^ _lsr(z, 31)


def h_t(seed: int, stream: int, idx):
    return splitmix64_t(idx ^ _i64(seed ^ (stream << 56)))


def mulhi_t(hv, m):
    """floor(hv * m / 2^64) for 0 <= m < 2^32 (m a Python int or an int64 tensor)."""
    lo = hv & 0xFFFFFFFF
    hi = _lsr(hv, 32)
    x = lo * m
    return _lsr(hi * m + _lsr(x, 32), 32)


def _u32_t(x):
    """int64 values in [0, 2^32) -> int32 tensor with the same 32 bits."""
    torch = _t()
    return (x - ((x >> 31) & 1) * (1 << 32)).to(torch.int32)


def raw_keys_t(seed: int, idx, alphabet: int | None = None):
    k = mulhi_t(h_t(seed, 0, idx), D)
    if alphabet is not None:
        k = k % alphabet
    return k


def updates_t(seed: int, start: int, count: int, delete_frac4: int = 1, device="cuda"):
    """updates() on a torch device: (keys int32, vals int32, is_delete uint8), the
    same bits as the numpy arrays."""
    torch = _t()
    idx = torch.arange(start, start + count, dtype=torch.int64, device=device)
    keys = raw_keys_t(seed, idx)
    vals = idx
    if delete_frac4 <= 0:
        return _u32_t(keys), _u32_t(vals & 0xFFFFFFFF), torch.zeros(count, dtype=torch.uint8,
                                                                   device=device)
    is_del = (h_t(seed, 1, idx) & 3) < delete_frac4  # % 4 of a uint64 = its low 2 bits
    safe = torch.clamp(idx, min=1)
    u = mulhi_t(h_t(seed, 2, idx), safe)
    tgt = raw_keys_t(seed, u)
    tgt = torch.where(idx == 0, keys, tgt)
    keys = torch.where(is_del, tgt, keys)
    vals = torch.where(is_del, torch.zeros_like(vals), vals & 0xFFFFFFFF)
    return _u32_t(keys), _u32_t(vals), is_del.to(torch.uint8)


def lookup_queries_t(seed: int, nq: int, n_updates: int, device="cuda"):
    torch = _t()
    j = torch.arange(nq, dtype=torch.int64, device=device)
    u = mulhi_t(h_t(seed, 4, j), max(n_updates, 1))
    hit = raw_keys_t(seed, u)
    fresh = mulhi_t(h_t(seed, 3, j), D)
    return _u32_t(torch.where((j & 1) == 0, hit, fresh))


def range_queries_t(seed: int, nq: int, n_resident: int, L: float, device="cuda"):
    torch = _t()
    w = max(1, int(round(L * D / max(n_resident, 1))))
    w = min(w, D)
    j = torch.arange(nq, dtype=torch.int64, device=device)
    k1 = mulhi_t(h_t(seed, 5, j), D - w + 1)
    k2 = k1 + (w - 1)
    return _u32_t(k1), _u32_t(k2)
