"""paper_1707_05354_b200 -- B200-native GPU LSM batched-update hot path.

Thin ctypes binding over the C ABI in include/gpulsm.h (libgpulsm.so, built
in-tree for sm_100a by paper_1707_05354_b200.build). Every step of the path
runs in the library's CUDA kernels; this module only marshals pointers,
sizes and the current torch CUDA stream. PyTorch provides device memory,
streams and process groups. There is no CPU fallback: if the library is
missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GPULSM_LIB selects another in-tree build of the same sources (A/B variants
# built by build.build_variant); default: libgpulsm.so
LIB_PATH = os.path.join(_HERE, os.environ.get("GPULSM_LIB", "libgpulsm.so"))

LSM_OK = 0
LSM_ERR_CAPACITY = 4
LSM_ERR_KEY_DOMAIN = 3
LSM_NOT_FOUND = 0xFFFFFFFF
LSM_PLACEBO = 0xFFFFFFFE
MAX_KEY = 0x7FFFFFFE
LSM_MAX_LEVELS = 40
KERNEL_CLASSES = ["sort_hist", "sort_pass", "merge", "lookup", "count", "range",
                  "scan", "cleanup", "other"]

_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_st = ctypes.c_int

# name -> (argtypes, restype); the exact entry points of include/gpulsm.h
SIGNATURES = {
    "lsm_create": ([_u64, ctypes.POINTER(_vp)], _st),
    "lsm_create_sa": ([_u64, ctypes.POINTER(_vp)], _st),
    "lsm_create_with_allocator": ([_u64, _vp, ctypes.POINTER(_vp)], _st),
    "lsm_is_sa": ([_vp, ctypes.POINTER(ctypes.c_int)], _st),
    "lsm_destroy": ([_vp], _st),
    "lsm_reserve": ([_vp, _u64, _vp], _st),
    "lsm_clear": ([_vp, _vp], _st),
    "lsm_update": ([_vp, _vp, _vp, _vp, _u64, _vp], _st),
    "lsm_update_records": ([_vp, _vp, _u64, _vp], _st),
    "lsm_insert": ([_vp, _vp, _vp, _u64, _vp], _st),
    "lsm_delete": ([_vp, _vp, _u64, _vp], _st),
    "lsm_update_host": ([_vp, _vp, _vp, _vp, _u64, _vp], _st),
    "lsm_lookup": ([_vp, _vp, _u64, _vp, _vp, _vp], _st),
    "lsm_lookup_host": ([_vp, _vp, _u64, _vp, _vp, _vp], _st),
    "lsm_count": ([_vp, _vp, _vp, _u64, _vp, _vp], _st),
    "lsm_bulk_build": ([_vp, _vp, _vp, _vp, _u64, _vp], _st),
    "lsm_update_batches": ([_vp, _vp, _vp, _vp, _u64, _vp], _st),
    "lsm_successor": ([_vp, _vp, _u64, _vp, _vp, _vp, _vp], _st),
    "lsm_predecessor": ([_vp, _vp, _u64, _vp, _vp, _vp, _vp], _st),
    "lsm_range": ([_vp, _vp, _vp, _u64, _vp, _vp, _vp, _u64, ctypes.POINTER(_u64), _vp], _st),
    "lsm_cleanup": ([_vp, _vp], _st),
    "lsm_batch_size": ([_vp, ctypes.POINTER(_u64)], _st),
    "lsm_num_batches": ([_vp, ctypes.POINTER(_u64)], _st),
    "lsm_query_levels": ([_vp, ctypes.POINTER(ctypes.c_uint32)], _st),
    "lsm_level_view": ([_vp, ctypes.c_uint32, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                        ctypes.POINTER(_u64)], _st),
    "lsm_sync": ([_vp, _vp], _st),
    "lsm_launch_count": ([_vp], _u64),
    "lsm_status_string": ([_st], ctypes.c_char_p),
    "lsm_profile_enable": ([_vp, ctypes.c_int], _st),
    "lsm_profile_read": ([_vp, _vp], _st),
    "lsm_shard_bucket": ([_vp, _vp, _vp, _vp, _u64, ctypes.c_uint32, ctypes.c_int, _vp, _vp, _vp,
                          _vp, _vp, _vp], _st),
    "lsm_shard_bucket_records": ([_vp, _vp, _vp, _vp, _u64, ctypes.c_uint32, _vp, _vp, _vp], _st),
    "lsm_shard_scatter": ([_vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp], _st),
    "lsm_nccl_unique_id": ([_vp], _st),
    "lsm_router_create": ([_vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _u64, _u64,
                           ctypes.POINTER(_vp)], _st),
    "lsm_router_update": ([_vp, _vp, _vp, _vp, _u64, _vp], _st),
    "lsm_router_flush": ([_vp, _vp], _st),
    "lsm_router_stats": ([_vp, ctypes.POINTER(_u64), ctypes.POINTER(_u64)], _st),
    "lsm_router_destroy": ([_vp], _st),
    "lsm_shard_route_ranges": ([_vp, _vp, _vp, _u64, ctypes.c_uint32, _vp, _vp, _vp, _u64,
                                ctypes.POINTER(_u64), _vp], _st),
    "lsm_shard_piece_sum": ([_vp, _vp, _vp, _vp, _u64, _u64, _vp, _vp], _st),
    "lsm_shard_piece_assemble": ([_vp, _vp, _vp, _vp, ctypes.c_uint32, _vp, _vp, _u64, _u64, _vp,
                                  _vp, _vp, _vp, _vp, _u64, ctypes.POINTER(_u64), _vp], _st),
    "lsm_shard_order_resolve": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_uint32,
                                 ctypes.c_int, _vp, _u64, _vp, _vp, _vp, _vp], _st),
}


class LsmProfile(ctypes.Structure):
    _fields_ = [("launches", _u64 * 9), ("ms", ctypes.c_double * 9),
                ("alg_bytes", ctypes.c_double * 9)]


class LsmError(RuntimeError):
    def __init__(self, code, what):
        self.code = code
        super().__init__(f"{what}: {status_string(code)} ({code})")


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libgpulsm.so (raises if absent -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"libgpulsm.so not built at {path}; run "
                              "`python -m paper_1707_05354_b200.build`")
        L = ctypes.CDLL(path)
        for name, (args, res) in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def status_string(code: int) -> str:
    return load_library().lsm_status_string(code).decode()


def _check(code, what):
    if code != LSM_OK:
        raise LsmError(code, what)


def _torch():
    import torch
    return torch


def _stream_ptr(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t, nbytes_per=4, name="tensor"):
    """Device pointer of a contiguous CUDA tensor with 4-byte (or 1-byte) items."""
    torch = _torch()
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.element_size() != nbytes_per:
        raise TypeError(f"{name} must have {nbytes_per}-byte elements, got {t.dtype}")
    return ctypes.c_void_p(t.data_ptr())


class _CudaView:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


def to_device(a, device="cuda"):
    """numpy u32/u8 array -> CUDA tensor of the same bytes (int32 / uint8)."""
    torch = _torch()
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).to(device)


def to_numpy_u32(t):
    return t.cpu().numpy().view(np.uint32)


# lsm_allocator (include/gpulsm.h): a stream-ordered allocator the library
# calls for its levels and scratch; GpuLSM(..., allocator="torch") passes
# torch's caching allocator.
_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class LsmAllocator(ctypes.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", ctypes.c_void_p)]


def _torch_allocator(device_index):
    torch = _torch()

    def alloc(nbytes, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device_index, int(stream or 0))
        except Exception:
            return None  # NULL: out of memory

    def free(p, stream, ctx):
        try:
            torch.cuda.caching_allocator_delete(int(p))
        except Exception:
            pass

    fa, ff = _ALLOC_FN(alloc), _FREE_FN(free)
    return LsmAllocator(fa, ff, None), (fa, ff)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for NativeRouter (created on one rank, broadcast)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.lsm_nccl_unique_id(buf), "lsm_nccl_unique_id")
    return buf.raw


class NativeRouter:
    """The native update router of the key-range sharded LSM (router.cu): bucket
    kernel + NCCL count exchange + one grouped NCCL exchange of encoded records
    + local insert, all enqueued from C++ on the caller's stream."""

    def __init__(self, local: "GpuLSM", nranks: int, rank: int, nccl_id: bytes, b_in: int,
                 b_local: int):
        self._lib = load_library()
        self.local = local
        h = ctypes.c_void_p()
        idb = ctypes.create_string_buffer(bytes(nccl_id), 128)
        _check(self._lib.lsm_router_create(local.h, int(nranks), int(rank), idb, int(b_in),
                                           int(b_local), ctypes.byref(h)), "lsm_router_create")
        self.h = h

    def update(self, keys, vals=None, is_delete=None, stream=None):
        _check(self._lib.lsm_router_update(self.h, _dev(keys, 4, "keys"), _dev(vals, 4, "vals"),
                                           _dev(is_delete, 1, "is_delete"), keys.numel(),
                                           _stream_ptr(stream)), "lsm_router_update")

    def flush(self, stream=None):
        _check(self._lib.lsm_router_flush(self.h, _stream_ptr(stream)), "lsm_router_flush")

    def stats(self):
        b, sp = _u64(0), _u64(0)
        _check(self._lib.lsm_router_stats(self.h, ctypes.byref(b), ctypes.byref(sp)),
               "lsm_router_stats")
        return int(b.value), int(sp.value)

    def close(self):
        if getattr(self, "h", None):
            self._lib.lsm_router_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GpuLSM:
    """A GPU LSM dictionary with batch size b on the current CUDA device.

    sa=True builds the paper's GPU SA comparison structure instead (N2: one
    sorted array, each batch merged into all of it; same calls)."""

    def __init__(self, b: int, reserve_batches: int = 0, sa: bool = False,
                 allocator: str | None = None):
        self._lib = load_library()
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("GpuLSM needs a CUDA device (no CPU fallback)")
        h = ctypes.c_void_p()
        if allocator == "torch":
            if sa:
                raise ValueError("allocator='torch' is for the LSM (not the SA) structure")
            self._alloc, self._alloc_keep = _torch_allocator(torch.cuda.current_device())
            _check(self._lib.lsm_create_with_allocator(int(b), ctypes.byref(self._alloc),
                                                       ctypes.byref(h)), "lsm_create_with_allocator")
        elif allocator is not None:
            raise ValueError("allocator must be None (the library's pool) or 'torch'")
        else:
            create = self._lib.lsm_create_sa if sa else self._lib.lsm_create
            _check(create(int(b), ctypes.byref(h)), "lsm_create_sa" if sa else "lsm_create")
        self.h = h
        self.b = int(b)
        self.sa = bool(sa)
        if reserve_batches:
            _check(self._lib.lsm_reserve(self.h, int(reserve_batches), _stream_ptr()),
                   "lsm_reserve")

    def close(self):
        if getattr(self, "h", None):
            self._lib.lsm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- updates ----
    def update(self, keys, vals=None, is_delete=None, stream=None):
        n = keys.numel()
        _check(self._lib.lsm_update(self.h, _dev(keys, 4, "keys"), _dev(vals, 4, "vals"),
                                    _dev(is_delete, 1, "is_delete"), n, _stream_ptr(stream)),
               "lsm_update")

    def update_records(self, records, stream=None):
        """A batch of encoded (key variable, value) records: int32 [n, 2]."""
        n = records.shape[0]
        _check(self._lib.lsm_update_records(self.h, _dev(records, 4, "records"), n,
                                            _stream_ptr(stream)), "lsm_update_records")

    def bulk_build(self, keys, vals=None, is_delete=None, stream=None):
        """N1 bulk build into an empty structure: all n elements form one batch,
        one sort, levels at the set bits of ceil(n/b)."""
        _check(self._lib.lsm_bulk_build(self.h, _dev(keys, 4, "keys"), _dev(vals, 4, "vals"),
                                        _dev(is_delete, 1, "is_delete"), keys.numel(),
                                        _stream_ptr(stream)), "lsm_bulk_build")

    def update_batches(self, keys, vals=None, is_delete=None, stream=None):
        """N1 multi-batch insertion: ceil(n/b) consecutive batches, oldest first,
        identical to that many update() calls (PAPER.md:860 footnote)."""
        _check(self._lib.lsm_update_batches(self.h, _dev(keys, 4, "keys"), _dev(vals, 4, "vals"),
                                            _dev(is_delete, 1, "is_delete"), keys.numel(),
                                            _stream_ptr(stream)), "lsm_update_batches")

    def insert(self, keys, vals, stream=None):
        _check(self._lib.lsm_insert(self.h, _dev(keys, 4, "keys"), _dev(vals, 4, "vals"),
                                    keys.numel(), _stream_ptr(stream)), "lsm_insert")

    def delete(self, keys, stream=None):
        _check(self._lib.lsm_delete(self.h, _dev(keys, 4, "keys"), keys.numel(),
                                    _stream_ptr(stream)), "lsm_delete")

    def update_host(self, keys: np.ndarray, vals=None, is_delete=None, stream=None):
        """lsm_update_host from (ideally pinned) host numpy/tensor buffers."""
        def hp(a):
            if a is None:
                return None
            if isinstance(a, np.ndarray):
                return ctypes.c_void_p(a.ctypes.data)
            return ctypes.c_void_p(a.data_ptr())
        n = len(keys)
        _check(self._lib.lsm_update_host(self.h, hp(keys), hp(vals), hp(is_delete), n,
                                         _stream_ptr(stream)), "lsm_update_host")

    # ---- queries ----
    def lookup(self, q, stream=None):
        torch = _torch()
        nq = q.numel()
        vals = torch.empty(nq, dtype=torch.int32, device=q.device)
        found = torch.empty(nq, dtype=torch.uint8, device=q.device)
        self.lookup_into(q, vals, found, stream)
        return vals, found

    def lookup_into(self, q, vals, found=None, stream=None):
        _check(self._lib.lsm_lookup(self.h, _dev(q, 4, "q"), q.numel(), _dev(vals, 4, "vals"),
                                    _dev(found, 1, "found"), _stream_ptr(stream)), "lsm_lookup")

    def lookup_host(self, q: np.ndarray, stream=None):
        q = np.ascontiguousarray(q, dtype=np.uint32)
        v = np.empty(len(q), np.uint32)
        f = np.empty(len(q), np.uint8)
        _check(self._lib.lsm_lookup_host(self.h, ctypes.c_void_p(q.ctypes.data), len(q),
                                         ctypes.c_void_p(v.ctypes.data),
                                         ctypes.c_void_p(f.ctypes.data), _stream_ptr(stream)),
               "lsm_lookup_host")
        return v, f

    def _order(self, fn, name, q, stream):
        torch = _torch()
        nq = q.numel()
        keys = torch.empty(nq, dtype=torch.int32, device=q.device)
        vals = torch.empty(nq, dtype=torch.int32, device=q.device)
        found = torch.empty(nq, dtype=torch.uint8, device=q.device)
        _check(fn(self.h, _dev(q, 4, "q"), nq, _dev(keys, 4, "keys"), _dev(vals, 4, "vals"),
                  _dev(found, 1, "found"), _stream_ptr(stream)), name)
        return keys, vals, found

    def successor(self, q, stream=None):
        """Smallest live key >= q per query (reading R23): (keys, vals, found)."""
        return self._order(self._lib.lsm_successor, "lsm_successor", q, stream)

    def predecessor(self, q, stream=None):
        """Largest live key <= q per query (reading R23): (keys, vals, found)."""
        return self._order(self._lib.lsm_predecessor, "lsm_predecessor", q, stream)

    def count(self, k1, k2, stream=None):
        torch = _torch()
        out = torch.empty(k1.numel(), dtype=torch.int32, device=k1.device)
        self.count_into(k1, k2, out, stream)
        return out

    def count_into(self, k1, k2, out, stream=None):
        if k1.numel() != k2.numel():
            raise ValueError("k1 and k2 differ in length")
        _check(self._lib.lsm_count(self.h, _dev(k1, 4, "k1"), _dev(k2, 4, "k2"), k1.numel(),
                                   _dev(out, 4, "out"), _stream_ptr(stream)), "lsm_count")

    def range(self, k1, k2, capacity: int | None = None, stream=None):
        """Returns (offsets[nq+1] int64, keys int32-bits, vals int32-bits)."""
        torch = _torch()
        nq = k1.numel()
        if k2.numel() != nq:
            raise ValueError("k1 and k2 differ in length")
        offsets = torch.empty(nq + 1, dtype=torch.int64, device=k1.device)
        cap = int(capacity) if capacity is not None else max(16, 16 * nq)
        while True:
            keys = torch.empty(max(cap, 1), dtype=torch.int32, device=k1.device)
            vals = torch.empty(max(cap, 1), dtype=torch.int32, device=k1.device)
            total = _u64(0)
            code = self._lib.lsm_range(self.h, _dev(k1, 4, "k1"), _dev(k2, 4, "k2"), nq,
                                       _dev(offsets, 8, "offsets"), _dev(keys, 4, "keys"),
                                       _dev(vals, 4, "vals"), cap, ctypes.byref(total),
                                       _stream_ptr(stream))
            if code == LSM_ERR_CAPACITY:
                cap = int(total.value)
                continue
            _check(code, "lsm_range")
            t = int(total.value)
            return offsets, keys[:t], vals[:t]

    def range_into(self, k1, k2, offsets, keys, vals, stream=None) -> int:
        total = _u64(0)
        _check(self._lib.lsm_range(self.h, _dev(k1, 4, "k1"), _dev(k2, 4, "k2"), k1.numel(),
                                   _dev(offsets, 8, "offsets"), _dev(keys, 4, "keys"),
                                   _dev(vals, 4, "vals"), keys.numel(), ctypes.byref(total),
                                   _stream_ptr(stream)), "lsm_range")
        return int(total.value)

    def cleanup(self, stream=None):
        _check(self._lib.lsm_cleanup(self.h, _stream_ptr(stream)), "lsm_cleanup")

    # ---- introspection ----
    @property
    def r(self) -> int:
        v = _u64(0)
        _check(self._lib.lsm_num_batches(self.h, ctypes.byref(v)), "lsm_num_batches")
        return int(v.value)

    @property
    def query_levels(self) -> int:
        """Sorted runs a query searches now (cleanup views count as one)."""
        v = ctypes.c_uint32()
        _check(self._lib.lsm_query_levels(self.h, ctypes.byref(v)), "lsm_query_levels")
        return int(v.value)

    def level(self, i: int):
        """(keys, vals) of level i as int32 CUDA tensors (copies; empty if level empty)."""
        torch = _torch()
        kp, vp, n = ctypes.c_void_p(), ctypes.c_void_p(), _u64(0)
        _check(self._lib.lsm_level_view(self.h, i, ctypes.byref(kp), ctypes.byref(vp),
                                        ctypes.byref(n)), "lsm_level_view")
        n = int(n.value)
        if n == 0:
            e = torch.empty(0, dtype=torch.int32, device="cuda")
            return e, e.clone()
        k = torch.as_tensor(_CudaView(kp.value, n, "<i4"), device="cuda").clone()
        v = torch.as_tensor(_CudaView(vp.value, n, "<i4"), device="cuda").clone()
        return k, v

    def sync(self, stream=None):
        _check(self._lib.lsm_sync(self.h, _stream_ptr(stream)), "lsm_sync")

    def clear(self, stream=None):
        _check(self._lib.lsm_clear(self.h, _stream_ptr(stream)), "lsm_clear")

    def reserve(self, max_batches: int, stream=None):
        _check(self._lib.lsm_reserve(self.h, int(max_batches), _stream_ptr(stream)),
               "lsm_reserve")

    # ---- key-range sharding kernels (used by sharded.ShardedLSM) ----
    def shard_bucket(self, keys, nshards, vals=None, ops=None, mode=0, want_perm=False,
                     stream=None):
        """Stable partition by owner shard -> (keys, vals, ops, perm, counts[P])."""
        torch = _torch()
        n = keys.numel()
        dev = keys.device
        ko = torch.empty(n, dtype=torch.int32, device=dev)
        vo = torch.empty(n, dtype=torch.int32, device=dev) if vals is not None else None
        oo = torch.empty(n, dtype=torch.uint8, device=dev) if ops is not None else None
        po = torch.empty(n, dtype=torch.int32, device=dev) if want_perm else None
        cnt = torch.empty(nshards, dtype=torch.int32, device=dev)
        _check(self._lib.lsm_shard_bucket(self.h, _dev(keys, 4, "keys"), _dev(vals, 4, "vals"),
                                          _dev(ops, 1, "ops"), n, nshards, mode, _dev(ko), _dev(vo),
                                          _dev(oo, 1), _dev(po), _dev(cnt), _stream_ptr(stream)),
               "lsm_shard_bucket")
        return ko, vo, oo, po, cnt

    def shard_bucket_records(self, keys, nshards, vals=None, ops=None, out=None, counts=None,
                             stream=None):
        """Range partition into encoded records -> (records int32 [n, 2], counts[P])."""
        torch = _torch()
        n = keys.numel()
        dev = keys.device
        rec = out if out is not None else torch.empty((n, 2), dtype=torch.int32, device=dev)
        cnt = counts if counts is not None else torch.empty(nshards, dtype=torch.int32, device=dev)
        _check(self._lib.lsm_shard_bucket_records(self.h, _dev(keys, 4, "keys"),
                                                  _dev(vals, 4, "vals"), _dev(ops, 1, "ops"), n,
                                                  nshards, _dev(rec), _dev(cnt),
                                                  _stream_ptr(stream)), "lsm_shard_bucket_records")
        return rec, cnt

    def shard_order_resolve(self, keys, vals, found, chunk_counts, ext_keys, ext_vals,
                            ext_found, nshards, last, perm, stream=None):
        """Owner-routed successor (last=False) / predecessor (last=True) answers in
        query order (see lsm_shard_order_resolve)."""
        torch = _torch()
        n = perm.numel()
        ko = torch.empty(n, dtype=torch.int32, device=perm.device)
        vo = torch.empty(n, dtype=torch.int32, device=perm.device)
        fo = torch.empty(n, dtype=torch.uint8, device=perm.device)
        _check(self._lib.lsm_shard_order_resolve(
            self.h, _dev(keys, 4, "keys"), _dev(vals, 4, "vals"), _dev(found, 1, "found"),
            _dev(chunk_counts, 4, "chunk_counts"), _dev(ext_keys, 4, "ext_keys"),
            _dev(ext_vals, 4, "ext_vals"), _dev(ext_found, 1, "ext_found"), int(nshards),
            int(bool(last)), _dev(perm, 4, "perm"), n, _dev(ko), _dev(vo), _dev(fo, 1),
            _stream_ptr(stream)), "lsm_shard_order_resolve")
        return ko, vo, fo

    def shard_scatter(self, perm, vals_in, found_in, vals_out, found_out, stream=None):
        _check(self._lib.lsm_shard_scatter(self.h, _dev(perm), _dev(vals_in), _dev(found_in, 1),
                                           perm.numel(), _dev(vals_out), _dev(found_out, 1),
                                           _stream_ptr(stream)), "lsm_shard_scatter")

    def shard_route_ranges(self, k1, k2, nshards, stream=None):
        """Pieces of the (k1, k2) queries on the shards they cover -> (pk1, pk2,
        pstart[nq+1] int32 (query q's pieces are [pstart[q], pstart[q+1])))."""
        torch = _torch()
        nq = k1.numel()
        dev = k1.device
        pstart = torch.empty(nq + 1, dtype=torch.int32, device=dev)
        cap = nq + 1024
        while True:
            pk1 = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            pk2 = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            npc = _u64(0)
            st = self._lib.lsm_shard_route_ranges(
                self.h, _dev(k1, 4, "k1"), _dev(k2, 4, "k2"), nq, int(nshards), _dev(pstart),
                _dev(pk1), _dev(pk2), cap, ctypes.byref(npc), _stream_ptr(stream))
            if st == LSM_ERR_CAPACITY and int(npc.value) > cap:
                cap = int(npc.value)
                continue
            _check(st, "lsm_shard_route_ranges")
            n = int(npc.value)
            return pk1[:n], pk2[:n], pstart

    def shard_piece_sum(self, counts_in, perm, pstart, nq, stream=None):
        """Per-query sums of piece counts (counts_in in bucket order)."""
        torch = _torch()
        out = torch.empty(nq, dtype=torch.int32, device=pstart.device)
        _check(self._lib.lsm_shard_piece_sum(self.h, _dev(counts_in), _dev(perm), _dev(pstart),
                                             int(nq), int(perm.numel()), _dev(out),
                                             _stream_ptr(stream)), "lsm_shard_piece_sum")
        return out

    def shard_piece_assemble(self, offs, block_len, chunk_counts, nshards, perm, pstart, nq,
                             keys_in, vals_in, stream=None):
        """Range answers from the shards' piece results: offs int64
        [npieces] (bucket order, each shard's own numbering), block_len int64
        [nshards], chunk_counts int32 [nshards] (pieces sent to each shard), the
        pair blocks concatenated in shard order -> (offsets[nq+1] int64, keys, vals)."""
        torch = _torch()
        dev = pstart.device
        cap = int(keys_in.numel())
        offsets = torch.empty(nq + 1, dtype=torch.int64, device=dev)
        keys = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        total = _u64(0)
        _check(self._lib.lsm_shard_piece_assemble(
            self.h, _dev(offs, 8, "offs"), _dev(block_len, 8, "block_len"),
            _dev(chunk_counts, 4, "chunk_counts"), int(nshards), _dev(perm, 4, "perm"),
            _dev(pstart, 4, "pstart"), int(nq), int(perm.numel()), _dev(keys_in, 4, "keys_in"),
            _dev(vals_in, 4, "vals_in"), _dev(offsets, 8, "offsets"), _dev(keys, 4, "keys"),
            _dev(vals, 4, "vals"), cap, ctypes.byref(total), _stream_ptr(stream)),
            "lsm_shard_piece_assemble")
        t = int(total.value)
        return offsets, keys[:t], vals[:t]

    @property
    def launch_count(self) -> int:
        return int(self._lib.lsm_launch_count(self.h))

    def profile_enable(self, on: bool = True):
        _check(self._lib.lsm_profile_enable(self.h, 1 if on else 0), "lsm_profile_enable")

    def profile_read(self) -> dict:
        p = LsmProfile()
        _check(self._lib.lsm_profile_read(self.h, ctypes.byref(p)), "lsm_profile_read")
        return {name: {"launches": int(p.launches[i]), "ms": float(p.ms[i]),
                       "alg_bytes": float(p.alg_bytes[i])}
                for i, name in enumerate(KERNEL_CLASSES)}
