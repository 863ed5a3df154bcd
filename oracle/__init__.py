"""CPU oracle for the GPU LSM hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. The product package
(paper_1707_05354_b200) never imports it and shares no code with it.

  O1  OracleDict  -- std::map dictionary definition (rules 1-6)
  S1  ShadowLSM   -- structural LSM, paper algorithm step by step (§3-§4)
  O0  BruteDict   -- literal history scan (oracle/brute.py), tiny inputs only

The C++ library is built by build() (g++, stdlib only).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .brute import BruteDict  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lsm_oracle.cpp")
_SRCS = [_SRC, os.path.join(_HERE, "exhaustive.cpp")]
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)
u8p = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f)
                                                 for f in _SRCS):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread",
                               "-o", _LIB, *_SRCS])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, u64 = ctypes.c_void_p, ctypes.c_uint64
        sig = {
            "o1_create": ([u64], vp), "o1_destroy": ([vp], None),
            "oracle_exhaustive": ([ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_uint32], ctypes.c_int64),
            "o1_apply_batch": ([vp, u32p, u32p, u8p, u64], None),
            "o1_lookup": ([vp, u32p, u64, u32p, u8p], None),
            "o1_count": ([vp, u32p, u32p, u64, u32p], None),
            "o1_successor": ([vp, u32p, u64, u32p, u32p, u8p], None),
            "o1_predecessor": ([vp, u32p, u64, u32p, u32p, u8p], None),
            "o1_range": ([vp, u32p, u32p, u64, u64p, u32p, u32p, u64], u64),
            "o1_bulk_build": ([vp, u32p, u32p, u8p, u64], None),
            "s1_bulk_build": ([vp, u32p, u32p, u8p, u64], ctypes.c_int),
            "sa_create": ([u64], vp), "sa_destroy": ([vp], None),
            "sa_update": ([vp, u32p, u32p, u8p, u64], None),
            "sa_bulk_build": ([vp, u32p, u32p, u8p, u64], ctypes.c_int),
            "sa_cleanup": ([vp], None), "sa_size": ([vp], u64),
            "sa_num_batches": ([vp], u64), "sa_merged_records": ([vp], u64),
            "sa_array": ([vp, u32p, u32p], None),
            "o1mt_create": ([u64, ctypes.c_uint32], vp), "o1mt_destroy": ([vp], None),
            "o1mt_apply_batch": ([vp, u32p, u32p, u8p, u64], None),
            "o1mt_lookup": ([vp, u32p, u64, u32p, u8p], None), "o1mt_size": ([vp], u64),
            "o1_cleanup": ([vp], None), "o1_size": ([vp], u64),
            "o1_num_batches": ([vp], u64), "o1_dump": ([vp, u32p, u32p], None),
            "s1_create": ([u64], vp), "s1_destroy": ([vp], None),
            "s1_update": ([vp, u32p, u32p, u8p, u64], None),
            "s1_cleanup": ([vp], None), "s1_num_batches": ([vp], u64),
            "s1_merged_records": ([vp], u64), "s1_domain_error": ([vp], ctypes.c_int),
            "s1_num_levels": ([vp], u64), "s1_level_size": ([vp, u64], u64),
            "s1_level": ([vp, u64, u32p, u32p, u64p], None),
            "s1_lookup": ([vp, u32p, u64, u32p, u8p], None),
            "s1_count": ([vp, u32p, u32p, u64, u32p, u64p], None),
            "s1_range": ([vp, u32p, u32p, u64, u64p, u32p, u32p, u64], u64),
            "s1_lower_bound": ([u32p, u64, ctypes.c_uint32], u64),
            "s1_upper_bound": ([u32p, u64, ctypes.c_uint32], u64),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _u8(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.uint8)


def lower_bound(packed, q):
    a = _u32(packed)
    return int(lib().s1_lower_bound(_p(a, u32p), len(a), int(q)))


def upper_bound(packed, q):
    a = _u32(packed)
    return int(lib().s1_upper_bound(_p(a, u32p), len(a), int(q)))


def dump_text(shadow) -> str:
    """SPEC.md:305-307 text format: `lsm b=<b> r=<r>` then one line per full
    level: `level <i>: <orig key>:<R|T>:<value> ...`."""
    lines = [f"lsm b={shadow.b} r={shadow.r}"]
    for i in range(shadow.num_levels()):
        k, v = shadow.level(i)
        if len(k) == 0:
            continue
        items = " ".join(f"{int(x) >> 1}:{'R' if int(x) & 1 else 'T'}:{int(y)}"
                         for x, y in zip(k, v))
        lines.append(f"level {i}: {items}")
    return "\n".join(lines)


class OracleDict:
    """O1: plain sequential ordered map under batch rules 1-6."""

    def __init__(self, b: int):
        self.b = b
        self.h = lib().o1_create(b)

    def __del__(self):
        if getattr(self, "h", None):
            lib().o1_destroy(self.h)
            self.h = None

    def apply_batch(self, keys, vals=None, is_delete=None):
        keys = _u32(keys)
        vals = _u32(vals) if vals is not None else np.zeros_like(keys)
        d = _u8(is_delete)
        lib().o1_apply_batch(self.h, _p(keys, u32p), _p(vals, u32p), _p(d, u8p), len(keys))

    def lookup(self, q):
        q = _u32(q)
        v = np.empty(len(q), np.uint32)
        f = np.empty(len(q), np.uint8)
        lib().o1_lookup(self.h, _p(q, u32p), len(q), _p(v, u32p), _p(f, u8p))
        return v, f

    def _order_query(self, fn, q):
        q = _u32(q)
        k = np.empty(len(q), np.uint32)
        v = np.empty(len(q), np.uint32)
        f = np.empty(len(q), np.uint8)
        fn(self.h, _p(q, u32p), len(q), _p(k, u32p), _p(v, u32p), _p(f, u8p))
        return k, v, f

    def successor(self, q):
        """Smallest live key >= q (R23): (keys, vals, found)."""
        return self._order_query(lib().o1_successor, q)

    def predecessor(self, q):
        """Largest live key <= q (R23): (keys, vals, found)."""
        return self._order_query(lib().o1_predecessor, q)

    def count(self, k1, k2):
        k1, k2 = _u32(k1), _u32(k2)
        out = np.empty(len(k1), np.uint32)
        lib().o1_count(self.h, _p(k1, u32p), _p(k2, u32p), len(k1), _p(out, u32p))
        return out

    def range(self, k1, k2):
        k1, k2 = _u32(k1), _u32(k2)
        nq = len(k1)
        off = np.empty(nq + 1, np.uint64)
        cap = int(self.count(k1, k2).astype(np.uint64).sum())
        ko = np.empty(max(cap, 1), np.uint32)
        vo = np.empty(max(cap, 1), np.uint32)
        tot = lib().o1_range(self.h, _p(k1, u32p), _p(k2, u32p), nq, _p(off, u64p),
                             _p(ko, u32p), _p(vo, u32p), cap)
        return off, ko[:tot], vo[:tot]

    def bulk_build(self, keys, vals=None, is_delete=None):
        """N1 (R24): all elements as one batch; r = ceil(n/b)."""
        keys = _u32(keys)
        vals = _u32(vals) if vals is not None else np.zeros_like(keys)
        d = _u8(is_delete)
        lib().o1_bulk_build(self.h, _p(keys, u32p), _p(vals, u32p), _p(d, u8p), len(keys))

    def cleanup(self):
        lib().o1_cleanup(self.h)

    @property
    def r(self):
        return int(lib().o1_num_batches(self.h))

    def __len__(self):
        return int(lib().o1_size(self.h))

    def items(self):
        n = len(self)
        k = np.empty(n, np.uint32)
        v = np.empty(n, np.uint32)
        if n:
            lib().o1_dump(self.h, _p(k, u32p), _p(v, u32p))
        return k, v


class ShadowLSM:
    """S1: the structural LSM of the paper (levels bit-exact)."""

    def __init__(self, b: int):
        self.b = b
        self.h = lib().s1_create(b)

    def __del__(self):
        if getattr(self, "h", None):
            lib().s1_destroy(self.h)
            self.h = None

    def update(self, keys, vals=None, is_delete=None):
        keys = _u32(keys)
        vals = _u32(vals) if vals is not None else np.zeros_like(keys)
        d = _u8(is_delete)
        lib().s1_update(self.h, _p(keys, u32p), _p(vals, u32p), _p(d, u8p), len(keys))

    def bulk_build(self, keys, vals=None, is_delete=None):
        """N1 bulk build (R24): one sort, sliced into levels."""
        keys = _u32(keys)
        vals = _u32(vals) if vals is not None else np.zeros_like(keys)
        d = _u8(is_delete)
        rc = lib().s1_bulk_build(self.h, _p(keys, u32p), _p(vals, u32p), _p(d, u8p), len(keys))
        if rc != 0:
            raise ValueError("bulk_build needs an empty structure and n >= 1")

    def cleanup(self):
        lib().s1_cleanup(self.h)

    @property
    def r(self):
        return int(lib().s1_num_batches(self.h))

    @property
    def merged_records(self):
        return int(lib().s1_merged_records(self.h))

    @property
    def domain_error(self):
        return bool(lib().s1_domain_error(self.h))

    def num_levels(self):
        return int(lib().s1_num_levels(self.h))

    def level(self, i, with_tags=False):
        n = int(lib().s1_level_size(self.h, i)) if i < self.num_levels() else 0
        k = np.empty(n, np.uint32)
        v = np.empty(n, np.uint32)
        t = np.empty(n, np.uint64) if with_tags else None
        if n:
            lib().s1_level(self.h, i, _p(k, u32p), _p(v, u32p), _p(t, u64p))
        return (k, v, t) if with_tags else (k, v)

    def lookup(self, q):
        q = _u32(q)
        v = np.empty(len(q), np.uint32)
        f = np.empty(len(q), np.uint8)
        lib().s1_lookup(self.h, _p(q, u32p), len(q), _p(v, u32p), _p(f, u8p))
        return v, f

    def count(self, k1, k2, return_candidates=False):
        k1, k2 = _u32(k1), _u32(k2)
        out = np.empty(len(k1), np.uint32)
        c = np.zeros(1, np.uint64)
        lib().s1_count(self.h, _p(k1, u32p), _p(k2, u32p), len(k1), _p(out, u32p), _p(c, u64p))
        return (out, int(c[0])) if return_candidates else out

    def range(self, k1, k2):
        k1, k2 = _u32(k1), _u32(k2)
        nq = len(k1)
        off = np.empty(nq + 1, np.uint64)
        cap = int(self.count(k1, k2).astype(np.uint64).sum())
        ko = np.empty(max(cap, 1), np.uint32)
        vo = np.empty(max(cap, 1), np.uint32)
        tot = lib().s1_range(self.h, _p(k1, u32p), _p(k2, u32p), nq, _p(off, u64p),
                             _p(ko, u32p), _p(vo, u32p), cap)
        return off, ko[:tot], vo[:tot]


class ShadowSA:
    """N2: the paper's GPU SA (one sorted array)."""

    def __init__(self, b: int):
        self.b = b
        self.h = lib().sa_create(b)

    def __del__(self):
        if getattr(self, "h", None):
            lib().sa_destroy(self.h)
            self.h = None

    def update(self, keys, vals=None, is_delete=None):
        keys = _u32(keys)
        vals = _u32(vals) if vals is not None else np.zeros_like(keys)
        d = _u8(is_delete)
        lib().sa_update(self.h, _p(keys, u32p), _p(vals, u32p), _p(d, u8p), len(keys))

    def bulk_build(self, keys, vals=None, is_delete=None):
        keys = _u32(keys)
        vals = _u32(vals) if vals is not None else np.zeros_like(keys)
        d = _u8(is_delete)
        if lib().sa_bulk_build(self.h, _p(keys, u32p), _p(vals, u32p), _p(d, u8p), len(keys)):
            raise ValueError("bulk_build needs an empty structure and n >= 1")

    def cleanup(self):
        lib().sa_cleanup(self.h)

    @property
    def r(self):
        return int(lib().sa_num_batches(self.h))

    @property
    def merged_records(self):
        return int(lib().sa_merged_records(self.h))

    def array(self):
        n = int(lib().sa_size(self.h))
        k = np.empty(n, np.uint32)
        v = np.empty(n, np.uint32)
        if n:
            lib().sa_array(self.h, _p(k, u32p), _p(v, u32p))
        return k, v


class ShardedOracleDict:
    """O1 over T key-range shards, one thread each (CPU-baseline timing only)."""

    def __init__(self, b: int, threads: int):
        self.threads = int(threads)
        self.h = lib().o1mt_create(b, self.threads)

    def __del__(self):
        if getattr(self, "h", None):
            lib().o1mt_destroy(self.h)
            self.h = None

    def apply_batch(self, keys, vals=None, is_delete=None):
        keys = _u32(keys)
        vals = _u32(vals) if vals is not None else np.zeros_like(keys)
        d = _u8(is_delete)
        lib().o1mt_apply_batch(self.h, _p(keys, u32p), _p(vals, u32p), _p(d, u8p), len(keys))

    def lookup(self, q):
        q = _u32(q)
        v = np.empty(len(q), np.uint32)
        f = np.empty(len(q), np.uint8)
        lib().o1mt_lookup(self.h, _p(q, u32p), len(q), _p(v, u32p), _p(f, u8p))
        return v, f

    def __len__(self):
        return int(lib().o1mt_size(self.h))


def exhaustive(b: int, nbatch: int, alphabet: int, threads: int = 0) -> int:
    """Every schedule of nbatch batches of b updates over `alphabet` keys x
    {insert, delete}: O0 (history scan) vs O1 vs S1 (oracle/exhaustive.cpp).
    Returns the number of schedules; raises on the first disagreement."""
    threads = threads or os.cpu_count() or 1
    r = int(lib().oracle_exhaustive(b, nbatch, alphabet, threads))
    if r < 0:
        raise AssertionError(f"oracle disagreement at schedule {-r - 1} (b={b}, nbatch={nbatch}, "
                             f"alphabet={alphabet})")
    return r

