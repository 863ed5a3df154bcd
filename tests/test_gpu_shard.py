"""GPU tests of the key-range sharding kernels (lsm_shard_*) and of the
sharded router on one GPU (NCCL, world size 1). Multi-rank routing logic is
covered on CPU by tests/test_sharded_gloo.py."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1707_05354_b200 as pkg  # noqa: E402
from paper_1707_05354_b200 import to_device, to_numpy_u32  # noqa: E402


def _owner(k, P, mode):
    k = k.astype(np.uint64)
    if mode == 0:
        return np.minimum((k * np.uint64(P)) >> np.uint64(31), P - 1).astype(np.int64)
    h = (k * np.uint64(0x9E3779B1)) & np.uint64(0xFFFFFFFF)
    bits = int(P).bit_length() - 1
    return (h >> np.uint64(32 - bits)).astype(np.int64) if bits else np.zeros(len(k), np.int64)


@pytest.mark.parametrize("P,mode,n", [(1, 0, 1000), (2, 0, 4097), (3, 0, 12345), (8, 0, 1 << 18),
                                      (64, 0, 50_000), (2, 1, 9999), (64, 1, 1 << 17), (8, 0, 0)])
def test_bucket_kernel_is_a_stable_partition(P, mode, n):
    g = pkg.GpuLSM(16)
    k = synth.uniform_u32(3, 6, n)
    k[: n // 10] &= 0x7FFFFFFF
    v = synth.uniform_u32(3, 7, n)
    o = (synth.uniform_u32(3, 8, n) & 1).astype(np.uint8)
    kb, vb, ob, pb, cnt = g.shard_bucket(
        to_device(k), P, vals=to_device(v), ops=to_device(o), mode=mode, want_perm=True)
    own = _owner(k, P, mode)
    perm = np.argsort(own, kind="stable")
    assert np.array_equal(to_numpy_u32(cnt), np.bincount(own, minlength=P).astype(np.uint32))
    assert np.array_equal(to_numpy_u32(kb), k[perm])
    assert np.array_equal(to_numpy_u32(vb), v[perm])
    assert np.array_equal(ob.cpu().numpy(), o[perm])
    assert np.array_equal(pb.cpu().numpy().astype(np.int64), perm)


def test_scatter_clip_sum_kernels():
    g = pkg.GpuLSM(16)
    n = 100_000
    perm = np.random.default_rng(1).permutation(n).astype(np.int32)
    vals = synth.uniform_u32(1, 1, n)
    found = (vals & 1).astype(np.uint8)
    vo = torch.empty(n, dtype=torch.int32, device="cuda")
    fo = torch.empty(n, dtype=torch.uint8, device="cuda")
    g.shard_scatter(to_device(perm), to_device(vals), to_device(found), vo, fo)
    ev = np.empty(n, np.uint32)
    ev[perm] = vals
    ef = np.empty(n, np.uint8)
    ef[perm] = found
    assert np.array_equal(to_numpy_u32(vo), ev) and np.array_equal(fo.cpu().numpy(), ef)
    k1 = synth.uniform_u32(2, 1, n)
    k2 = synth.uniform_u32(2, 2, n)
    lo, hi = 1 << 29, (1 << 30) - 1
    c1, c2 = g.shard_clip(to_device(k1), to_device(k2), lo, hi)
    a, z = k1.astype(np.int64), k2.astype(np.int64)
    empty = (a > z) | (z < lo) | (a > hi)
    assert np.array_equal(to_numpy_u32(c1), np.where(empty, 1, np.maximum(a, lo)).astype(np.uint32))
    assert np.array_equal(to_numpy_u32(c2), np.where(empty, 0, np.minimum(z, hi)).astype(np.uint32))
    parts = (synth.uniform_u32(4, 1, 3 * n) >> 8).astype(np.uint32)
    s = g.shard_sum(to_device(parts), 3, n)
    assert np.array_equal(to_numpy_u32(s), parts.reshape(3, n).sum(axis=0).astype(np.uint32))


def test_range_assemble_kernel():
    # lsm_shard_range_assemble vs a numpy definition: P = 3 shards' parts for
    # nq queries, offsets slices in the senders' numbering, blocks in shard
    # order; each query's pieces concatenated shard 0 first.
    g = pkg.GpuLSM(16)
    rng = np.random.default_rng(4)
    P, nq = 3, 5000
    cnt = rng.integers(0, 6, (P, nq))
    cnt[:, 7] = 0  # a query with nothing anywhere
    offs = np.zeros((P, nq), np.int64)
    blen = cnt.sum(axis=1)
    for s_ in range(P):
        start = int(rng.integers(0, 1000))  # sender numbering need not start at 0
        offs[s_] = start + np.concatenate([[0], np.cumsum(cnt[s_])[:-1]])
    tot = int(blen.sum())
    keys = rng.integers(0, 1 << 31, tot).astype(np.uint32)
    vals = np.arange(tot, dtype=np.uint32)
    o, k, v = g.shard_range_assemble(torch.from_numpy(offs.reshape(-1)).cuda(),
                                     torch.from_numpy(blen.astype(np.int64)).cuda(), P, nq,
                                     to_device(keys), to_device(vals))
    eoff = np.concatenate([[0], np.cumsum(cnt.sum(axis=0))])
    base = np.concatenate([[0], np.cumsum(blen)])
    ek, ev = [], []
    for q in range(nq):
        for s_ in range(P):
            src = base[s_] + offs[s_, q] - offs[s_, 0]
            ek.append(keys[src:src + cnt[s_, q]])
            ev.append(vals[src:src + cnt[s_, q]])
    assert np.array_equal(o.cpu().numpy(), eoff)
    assert np.array_equal(to_numpy_u32(k), np.concatenate(ek))
    assert np.array_equal(to_numpy_u32(v), np.concatenate(ev))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("native", [True, False])
def test_sharded_router_single_gpu_nccl(native):
    # native=True: the per-batch update path in router.cu (NCCL from C++);
    # False: the Python router (torch.distributed all-to-alls)
    import torch.distributed as dist
    from paper_1707_05354_b200.sharded import ShardedLSM
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        b = 1 << 14
        sh = ShardedLSM(b, native=native)
        assert (sh._native is not None) == native
        o = oracle.OracleDict(b)
        for j in range(9):
            k, v, d = synth.updates(5, j * b, b, delete_frac4=1, alphabet=50_000)
            sh.update(to_device(k), to_device(v), to_device(d))
            o.apply_batch(k, v, d)
        q = synth.lookup_queries(6, 20_000, 9 * b, alphabet=50_000)
        qv, qf = sh.lookup(to_device(q))
        ov, of = o.lookup(q)
        assert np.array_equal(qf.cpu().numpy(), of)
        assert np.array_equal(to_numpy_u32(qv), ov)
        k1, k2 = synth.range_queries(7, 3000, 9 * b, 12, domain=50_002)
        c = sh.count(to_device(k1), to_device(k2))
        assert np.array_equal(to_numpy_u32(c), o.count(k1, k2))
        for fn, ofn in ((sh.successor, o.successor), (sh.predecessor, o.predecessor)):
            gk, gv, gf = fn(to_device(q))
            ek, ev, ef = ofn(q)
            assert np.array_equal(gf.cpu().numpy(), ef)
            assert np.array_equal(to_numpy_u32(gk), ek) and np.array_equal(to_numpy_u32(gv), ev)
        ro, rk, rv = sh.range(to_device(k1), to_device(k2))
        ooff, ok, ov2 = o.range(k1, k2)
        assert np.array_equal(ro.cpu().numpy().astype(np.uint64), ooff)
        assert np.array_equal(to_numpy_u32(rk), ok) and np.array_equal(to_numpy_u32(rv), ov2)
    finally:
        dist.destroy_process_group()


def test_native_router_oversize_split():
    # b_local < b_in: every received batch exceeds the local batch size and is
    # split by a hash of the original key (equal keys stay together) into
    # sub-batches inserted in order -- lookups and counts equal to O1
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        b_in, b_local = 1 << 14, 3 << 12
        local = pkg.GpuLSM(b_local)
        rt = pkg.NativeRouter(local, 1, 0, pkg.nccl_unique_id(), b_in, b_local)
        o = oracle.OracleDict(b_in)
        for j in range(5):
            k, v, d = synth.updates(8, j * b_in, b_in, delete_frac4=1, alphabet=40_000)
            rt.update(to_device(k), to_device(v), to_device(d))
            o.apply_batch(k, v, d)
        rt.flush()
        assert rt.stats() == (5, 5)
        q = synth.lookup_queries(9, 20_000, 5 * b_in, alphabet=40_000)
        qv, qf = local.lookup(to_device(q))
        ov, of = o.lookup(q)
        assert np.array_equal(qf.cpu().numpy(), of) and np.array_equal(to_numpy_u32(qv), ov)
        k1, k2 = synth.range_queries(10, 3000, 5 * b_in, 12, domain=40_002)
        assert np.array_equal(to_numpy_u32(local.count(to_device(k1), to_device(k2))),
                              o.count(k1, k2))
        rt.close()
    finally:
        dist.destroy_process_group()
