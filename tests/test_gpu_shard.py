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


def test_scatter_kernel():
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


def _routing_queries(n, seed):
    # short ranges, ranges across shard boundaries, the whole query space,
    # empty ones (k1 > k2), keys above the domain (R8)
    k1 = synth.uniform_u32(seed, 1, n)
    w = (synth.uniform_u32(seed, 2, n) >> np.uint32(20 + seed % 3 * 3)).astype(np.uint64)
    k2 = np.minimum(k1.astype(np.uint64) + w, 0xFFFFFFFF).astype(np.uint32)
    k1[::13] = 0
    k2[::17] = 0xFFFFFFFF
    sel = np.arange(5, n, 19)
    sel = sel[k1[sel] > 0]
    k2[sel] = k1[sel] - 1  # empty: k1 > k2
    return k1, k2


@pytest.mark.parametrize("P", [1, 2, 3, 8, 64])
def test_route_and_piece_kernels(P):
    # lsm_shard_route_ranges / piece_sum / piece_assemble vs the numpy
    # stand-ins of the gloo tests' CPU backend (an independent implementation)
    from tests.test_sharded_gloo import CpuTestBackend
    cpu = CpuTestBackend(16)
    g = pkg.GpuLSM(16)
    n = 3000
    k1, k2 = _routing_queries(n, P)
    t1 = torch.from_numpy(k1.view(np.int32).copy())
    t2 = torch.from_numpy(k2.view(np.int32).copy())
    pk1, pk2, pstart = g.shard_route_ranges(t1.cuda(), t2.cuda(), P)
    ck1, ck2, cps = cpu.route_ranges(t1, t2, P)
    assert np.array_equal(pstart.cpu().numpy(), cps.numpy())
    assert np.array_equal(pk1.cpu().numpy(), ck1.numpy())
    assert np.array_equal(pk2.cpu().numpy(), ck2.numpy())
    npc = pk1.numel()
    assert npc > n // 2
    # pieces bucketed by owner; made-up per-piece answers from the owners
    _, _, _, perm, cnt = g.shard_bucket(pk1, P, vals=pk2, want_perm=True)
    rng = np.random.default_rng(P)
    pc = rng.integers(0, 7, npc).astype(np.int32)  # answers in bucket order
    s = g.shard_piece_sum(torch.from_numpy(pc).cuda(), perm, pstart, n)
    es = cpu.piece_sum(torch.from_numpy(pc), perm.cpu(), cps, n)
    assert np.array_equal(s.cpu().numpy(), es.numpy())
    # each owner numbers its output from an arbitrary start
    chunk = cnt.cpu().numpy().astype(np.int64)
    cstart = np.concatenate([[0], np.cumsum(chunk)])
    offs = np.zeros(npc, np.int64)
    blen = np.zeros(P, np.int64)
    for c in range(P):
        seg = pc[cstart[c]:cstart[c + 1]].astype(np.int64)
        if len(seg):
            offs[cstart[c]:cstart[c + 1]] = int(rng.integers(0, 1000)) + np.concatenate(
                [[0], np.cumsum(seg)[:-1]])
        blen[c] = seg.sum()
    tot = int(blen.sum())
    keys = rng.integers(0, 1 << 31, tot).astype(np.uint32)
    vals = np.arange(tot, dtype=np.uint32)
    args = [torch.from_numpy(offs), torch.from_numpy(blen), cnt.cpu(), P, perm.cpu(), cps, n,
            torch.from_numpy(keys.view(np.int32)), torch.from_numpy(vals.view(np.int32))]
    eo, ek, ev = cpu.piece_assemble(*args)
    o, k, v = g.shard_piece_assemble(*[a.cuda() if isinstance(a, torch.Tensor) else a for a in args])
    assert np.array_equal(o.cpu().numpy(), eo.numpy())
    assert np.array_equal(k.cpu().numpy(), ek.numpy())
    assert np.array_equal(v.cpu().numpy(), ev.numpy())


@pytest.mark.parametrize("P", [1, 3, 8])
def test_order_resolve_kernel(P):
    # lsm_shard_order_resolve vs the numpy stand-in of the gloo tests: owners'
    # local answers in bucket order, empty shards, queries no shard can answer
    from tests.test_sharded_gloo import CpuTestBackend
    cpu = CpuTestBackend(16)
    g = pkg.GpuLSM(16)
    rng = np.random.default_rng(P)
    n = 5000
    chunk = rng.multinomial(n, [1.0 / P] * P).astype(np.int32)
    k = rng.integers(0, 1 << 31, n).astype(np.int32)
    v = rng.integers(0, 1 << 31, n).astype(np.int32)
    f = (rng.random(n) < 0.6).astype(np.uint8)
    ek = rng.integers(0, 1 << 31, P).astype(np.int32)
    ev = rng.integers(0, 1 << 31, P).astype(np.int32)
    ef = (rng.random(P) < 0.5).astype(np.uint8)
    perm = rng.permutation(n).astype(np.int32)
    for last in (False, True):
        args = [torch.from_numpy(x) for x in (k, v, f, chunk, ek, ev, ef)] + [P, last,
                                                                         torch.from_numpy(perm)]
        eo = cpu.order_resolve(*args)
        go = g.shard_order_resolve(*[a.cuda() if isinstance(a, torch.Tensor) else a for a in args])
        for x, y in zip(go, eo):
            assert np.array_equal(x.cpu().numpy(), y.numpy()), (P, last)


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
