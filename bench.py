#!/usr/bin/env python3
"""bench.py -- GPU LSM hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

Workload (N=1): BASELINE.json configs[2] ("C3"): b = 2^20, 64 mixed batches
(75% insert / 25% delete) from empty -> 2^26 resident records, then 2^24
lookups (50% hit), 2^24 counts and 2^24 ranges at expected length L = 8,
cleanup, and the same queries again. One STEP = that whole cycle (every row of
SURVEY.md §8(a)). `value` = M updates/s over the update phase of the timed
steps (device time, CUDA events); the query and cleanup rates are reported in
`queries` / `cleanup`. Inputs (600 MB of updates, 512 MB structure) exceed
the 126 MB L2, so no explicit flush is needed.

N > 1: the key-range sharded LSM (paper_1707_05354_b200.sharded): the global
batch b_global = N * 2^20 is generated across ranks, routed to key owners by
the bucket kernel + NCCL all-to-all, and inserted into each rank's LSM.
Weak scaling; timing is the max over ranks.

--impl reference: the CPU oracle (oracle/, std::map) on the same config,
bounded samples per step (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

B = 1 << 20
R = 64
NQ = 1 << 24
L_RANGE = 8
METRIC = "M updates/s at batch b; M lookup/count/range queries/s; HBM GB/s vs peak"
UNIT = "M updates/s"
WORKLOAD = ("C3: b=2^20, 64 mixed batches (75% insert/25% delete) from empty -> 2^26 "
            "resident; 2^24 lookups (50% hit), 2^24 count + 2^24 range at L=8, before "
            "and after lsm_cleanup")


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clocks + throttle reasons with NVML during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting"}

    def __init__(self, index=0):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.hdl = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.hdl, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.hdl, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.hdl)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_baseline_oracle(seconds_budget=15.0):
    """The oracle O1 on a bounded sample of C3: key-range sharded
    over all host cores (the reported value) -- the first 56 batches are applied
    untimed so the timed last 8 batches go into a map of ~2^25.6 live keys, as
    on the GPU -- and the plain 1-thread std::map on the first batches (a
    near-empty map: an upper bound for its rate), under single_thread."""
    import oracle
    seed = synth.SEED_BASE + 2
    threads = os.cpu_count() or 1
    o = oracle.ShardedOracleDict(B, threads)
    t0 = time.perf_counter()
    for j in range(R - 8):
        o.apply_batch(*synth.updates(seed, j * B, B, delete_frac4=1))
    prefill_s = time.perf_counter() - t0
    tail = [synth.updates(seed, j * B, B, delete_frac4=1) for j in range(R - 8, R)]
    t0 = time.perf_counter()
    for k, v, d in tail:
        o.apply_batch(k, v, d)
    t_upd = time.perf_counter() - t0
    q = synth.lookup_queries(seed, 1 << 20, R * B)
    t1 = time.perf_counter()
    o.lookup(q)
    lk = (1 << 20) / (time.perf_counter() - t1) / 1e6
    resident = len(o)
    del o
    one = oracle.OracleDict(B)
    nb1 = 0
    t0 = time.perf_counter()
    for j in range(8):
        one.apply_batch(*synth.updates(seed, j * B, B, delete_frac4=1))
        nb1 += 1
        if time.perf_counter() - t0 > seconds_budget * 0.3:
            break
    upd_1 = nb1 * B / (time.perf_counter() - t0) / 1e6
    return {"value": 8 * B / t_upd / 1e6, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"C3 batches 57..64 (8x2^20 mixed updates) into {threads} key-range std::map "
                      f"shards (one thread each) already holding batches 1..56 (untimed, "
                      f"{prefill_s:.1f} s); then 2^20 lookups on the {resident} live keys",
            "lookup_mqps": lk, "resident_after": resident,
            "single_thread": {"value": upd_1, "cores": 1, "batches": nb1,
                              "sample": "first C3 batches into one empty std::map"}}


PARITY_LO, PARITY_HI = 5 << 25, 6 << 25  # 1/64 of the key domain


def check_queries(o1, lo, hi, q=None, lv=None, lf=None, k1=None, k2=None, cnt=None,
                  roff=None, rk=None, rv=None):
    """Compare one structure's query outputs with O1 on the key sub-range [lo, hi):
    O1 was fed only the updates whose key lies in [lo, hi) -- keys never interact
    (PAPER.md:94-110), so it answers every query inside the interval exactly. For
    range, the offsets of ALL queries must be the exclusive scan of the counts
    (count == len(range)). Returns (failures, numbers checked)."""
    from paper_1707_05354_b200 import to_numpy_u32
    fails, n = [], {}
    if q is not None:
        gv, gf = to_numpy_u32(lv), lf.cpu().numpy()
        sel = (q >= lo) & (q < hi)
        ov, of = o1.lookup(q[sel])
        if not (np.array_equal(gf[sel], of) and np.array_equal(gv[sel], ov)):
            fails.append("lookup")
        n["lookups"] = int(sel.sum())
    if k1 is not None and cnt is not None:
        gc = to_numpy_u32(cnt)
        ins = (k1 >= lo) & (k2 < hi) & (k1 <= k2)
        if not np.array_equal(gc[ins], o1.count(k1[ins], k2[ins])):
            fails.append("count")
        n["counts"] = int(ins.sum())
        if roff is not None:
            off = roff.cpu().numpy().astype(np.uint64)
            if off[0] != 0 or not np.array_equal(np.diff(off), gc.astype(np.uint64)):
                fails.append("range offsets != exclusive scan of counts")
            idx = np.nonzero(ins)[0]
            ooff, oks, ovs = o1.range(k1[idx], k2[idx])
            lens = np.diff(ooff).astype(np.int64)
            pos = np.repeat(off[idx].astype(np.int64), lens) + (
                np.arange(int(lens.sum())) - np.repeat(ooff[:-1].astype(np.int64), lens))
            pos_t = torch_index(pos, rk.device)
            if not (np.array_equal(to_numpy_u32(rk[pos_t]), oks) and
                    np.array_equal(to_numpy_u32(rv[pos_t]), ovs)):
                fails.append("range pairs")
            n["ranges"] = int(ins.sum())
            n["pairs"] = int(lens.sum())
            n["all_offsets_checked"] = len(off)
    return fails, n


def parity_gate(lsm, sub, q, k1, k2, lv, lf, cnt, roff, rk, rv, tot_pre, tot_post):
    """Check the timed step's outputs against the oracle before any number is
    printed: every lookup / count / range of the step inside the key sub-range
    (check_queries), the range totals before and after cleanup, and the
    post-cleanup level image restricted to the interval against O1's live
    pairs (R12). Exits non-zero on a mismatch: no timing line is emitted
    (S:477)."""
    import oracle
    from paper_1707_05354_b200 import to_numpy_u32
    lo, hi = PARITY_LO, PARITY_HI
    o1 = oracle.OracleDict(B)
    for k, v, d in sub:
        o1.apply_batch(k, v, d)
    o1.cleanup()
    fails, n = check_queries(o1, lo, hi, q, lv, lf, k1, k2, cnt, roff, rk, rv)
    off_last = int(roff[-1].item())
    if not (tot_pre == tot_post == off_last):
        fails.append("range totals before/after cleanup")
    # post-cleanup image inside [lo, hi): the encoded live pairs of O1
    ik, iv = [], []
    for i in range(lsm.r.bit_length()):
        kk, vv = lsm.level(i)
        kk, vv = to_numpy_u32(kk), to_numpy_u32(vv)
        m = ((kk >> 1) >= lo) & ((kk >> 1) < hi)
        ik.append(kk[m])
        iv.append(vv[m])
    ok_, ov_ = o1.items()
    if not (np.array_equal(np.concatenate(ik), (ok_ << 1) | 1) and
            np.array_equal(np.concatenate(iv), ov_)):
        fails.append("post-cleanup level image")
    if fails:
        sys.stderr.write(f"PARITY FAILED: {fails}\n")
        sys.exit(3)
    n.update({"ok": True, "oracle": "O1 (std::map) on the key sub-range [5*2^25, 6*2^25)",
              "live_pairs_in_image": int(len(ok_))})
    return n


def gate(name, fails):
    """Secondary configurations are parity-gated too: a mismatch ends the run."""
    if fails:
        sys.stderr.write(f"PARITY FAILED ({name}): {fails}\n")
        sys.exit(3)


def torch_index(pos, device):
    import torch
    return torch.from_numpy(pos).to(device)


# ---------------------------------------------------------------------------
# Secondary configurations; each parity-gated against
# O1 on the key sub-range [PARITY_LO, PARITY_HI). Reported under "secondary".
# ---------------------------------------------------------------------------

def _ev_timer(stream):
    import torch

    def timed(fn, reps=3):
        fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))
    return timed


def _queries(lsm, dev, q, k1, k2, timed, cap_factor=1.3):
    """lookup / count / range of the given queries (device tensors), timed;
    returns (rates, output tensors)."""
    import torch
    nq = q.numel()
    lv = torch.empty(nq, dtype=torch.int32, device=dev)
    lf = torch.empty(nq, dtype=torch.uint8, device=dev)
    nr = k1.numel()
    cnt = torch.empty(nr, dtype=torch.int32, device=dev)
    t_l = timed(lambda: lsm.lookup_into(q, lv, lf))
    t_c = timed(lambda: lsm.count_into(k1, k2, cnt))
    total = int(cnt.to(torch.int64).sum().item())
    roff = torch.empty(nr + 1, dtype=torch.int64, device=dev)
    rk = torch.empty(max(16, total + 16), dtype=torch.int32, device=dev)
    rv = torch.empty(max(16, total + 16), dtype=torch.int32, device=dev)
    got = []
    t_r = timed(lambda: got.append(lsm.range_into(k1, k2, roff, rk, rv)))
    rates = {"lookup_mqps": nq / (t_l * 1e-3) / 1e6, "count_mqps": nr / (t_c * 1e-3) / 1e6,
             "range_mqps": nr / (t_r * 1e-3) / 1e6, "pairs_per_range": total / max(nr, 1),
             "count_eq_len_range": got[-1] == total}
    return rates, (lv, lf, cnt, roff, rk, rv)


def _sub_oracle(b):
    import oracle
    return oracle.OracleDict(b)


def extra_c2(pkg, dev, stream):
    """C2 (BASELINE configs[1]; Table II protocol):
    b = 2^16 insert-only, 64 batches from empty; every batch's insert time
    (CUDA events around each lsm_update) -> min / max / harmonic mean rate
    over r (R17); at r in {1, 3, 7, 15, 31, 63, 64}: nq = n lookups (50 %
    hit), counts and ranges at L = 8."""
    import torch
    from paper_1707_05354_b200 import to_device
    b, R2 = 1 << 16, 64
    seed = synth.SEED_BASE + 1
    timed = _ev_timer(stream)
    data = [synth.updates(seed, j * b, b, delete_frac4=0) for j in range(R2)]
    dd = [(to_device(k, dev), to_device(v, dev), to_device(d, dev)) for k, v, d in data]
    lsm = pkg.GpuLSM(b, reserve_batches=R2)
    o1 = _sub_oracle(b)
    # (1) timing pass: the 64 inserts back to back, an event pair around each
    for _ in range(2):  # warm-up cycles (pool allocations, index storage)
        lsm.clear()
        for j in range(R2):
            lsm.update(*dd[j])
    lsm.clear()
    torch.cuda.synchronize()
    per = []
    for j in range(R2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lsm.update(*dd[j])
        e1.record(stream)
        per.append((e0, e1))
    torch.cuda.synchronize()
    # (2) query pass: the same inserts again, queries at the Table II-IV
    #     occupancies, O1 fed alongside
    lsm.clear()
    rows = []
    for j in range(R2):
        lsm.update(*dd[j])
        k, v, d = data[j]
        m = (k >= PARITY_LO) & (k < PARITY_HI)
        o1.apply_batch(k[m], v[m], d[m])
        r = j + 1
        if r in (1, 3, 7, 15, 31, 63, 64):
            n = r * b
            q = synth.lookup_queries(seed, n, n)
            k1, k2 = synth.range_queries(seed, n, n, 8)
            rates, outs = _queries(lsm, dev, to_device(q, dev), to_device(k1, dev),
                                   to_device(k2, dev), timed)
            fails, _ = check_queries(o1, PARITY_LO, PARITY_HI, q, outs[0], outs[1], k1, k2,
                                     outs[2], outs[3], outs[4], outs[5])
            gate(f"C2 r={r}", fails + ([] if rates["count_eq_len_range"] else ["count != len(range)"]))
            rows.append({"r": r, "levels": bin(r).count("1"), "nq": n, **rates})
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(e) for a, e in per])
    rate = b / (ms * 1e-3) / 1e6
    lsm.close()
    return {"workload": "C2: b=2^16 insert-only, 64 batches from empty; queries nq=n at L=8",
            "insert_mups": {"min": float(rate.min()), "max": float(rate.max()),
                            "harmonic_mean": float(R2 * b / (ms.sum() * 1e-3) / 1e6),
                            "min_at_r": int(np.argmin(rate)), "max_at_r": int(np.argmax(rate))},
            "timing": "CUDA events around each lsm_update (per-batch, Table II protocol)",
            "queries": rows, "parity": "O1 on the key sub-range, every checked r"}


def extra_c3p_sa_bulk(pkg, dev, stream, keys_d, vals_d, ops_d, sub, q, k1, k2):
    """C3' (§5.4 shape): 63 mixed batches of 2^20 (six
    occupied levels), queries, a multi-level cleanup (elem/s, GB/s), queries;
    N2: the GPU SA fed the same 63 batches, LSM-vs-SA
    ratios; N1: bulk build of all 64 C3 batches (2^26
    elements) into an empty LSM."""
    import torch
    from paper_1707_05354_b200 import to_device
    timed = _ev_timer(stream)
    R3 = 63
    dq, dk1, dk2 = to_device(q, dev), to_device(k1, dev), to_device(k2, dev)
    o1 = _sub_oracle(B)
    for k, v, d in sub[:R3]:
        o1.apply_batch(k, v, d)
    out = {}
    for name, sa in (("lsm", False), ("sa", True)):
        st = pkg.GpuLSM(B, reserve_batches=R, sa=sa)
        for _ in range(1):  # warm-up
            st.clear()
            for j in range(8):
                st.update(keys_d[j], vals_d[j], ops_d[j])
        st.clear()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for j in range(R3):
            st.update(keys_d[j], vals_d[j], ops_d[j])
        e1.record(stream)
        torch.cuda.synchronize()
        upd_ms = e0.elapsed_time(e1)
        rates, outs = _queries(st, dev, dq, dk1, dk2, timed)
        fails, _ = check_queries(o1, PARITY_LO, PARITY_HI, q, outs[0], outs[1], k1, k2, *outs[2:])
        gate(f"C3' {name} r=63", fails)
        res = {"update_mups": R3 * B / (upd_ms * 1e-3) / 1e6, "update_ms": upd_ms,
               "levels": bin(R3).count("1") if not sa else 1, **rates}
        if not sa:
            n = R3 * B
            # the first cleanup of a handle allocates its merge and compaction
            # buffers: run one untimed, then rebuild r = 63 and time the next
            st.cleanup()
            st.clear()
            for j in range(R3):
                st.update(keys_d[j], vals_d[j], ops_d[j])
            torch.cuda.synchronize()
            e0.record(stream)
            st.cleanup()
            e1.record(stream)
            torch.cuda.synchronize()
            c_ms = e0.elapsed_time(e1)
            r2 = st.r
            rates2, outs2 = _queries(st, dev, dq, dk1, dk2, timed)
            o1.cleanup()
            fails, _ = check_queries(o1, PARITY_LO, PARITY_HI, q, outs2[0], outs2[1], k1, k2,
                                     *outs2[2:])
            gate("C3' after cleanup", fails)
            res["cleanup"] = {"ms": c_ms, "melem_per_s": n / (c_ms * 1e-3) / 1e6,
                              "alg_GBps": (8.0 * n + 8.0 * r2 * B) / (c_ms * 1e-3) / 1e9,
                              "levels_merged": bin(R3).count("1"), "r_after": r2,
                              "stale_fraction": 1.0 - (len(o1) * 64.0) / n if len(o1) else None,
                              "note": "stale_fraction estimated from the 1/64 key sub-range"}
            res["after_cleanup"] = {**rates2, "levels": bin(r2).count("1")}
        st.close()
        out[name] = res
    L, S = out["lsm"], out["sa"]
    out["lsm_over_sa"] = {"updates": L["update_mups"] / S["update_mups"],
                          "lookup": L["lookup_mqps"] / S["lookup_mqps"],
                          "count": L["count_mqps"] / S["count_mqps"],
                          "range": L["range_mqps"] / S["range_mqps"],
                          "paper_K40c": "updates 13.5x; lookups 1/1.75; count/range 1/1.36-1/1.84 "
                                        "(PAPER.md:846, 946, 979-980; other b and n)"}
    # N1 bulk build: the 64 C3 batches as one input of 2^26 elements
    allk = torch.cat(keys_d)
    allv = torch.cat(vals_d)
    allo = torch.cat(ops_d)
    bl = pkg.GpuLSM(B)
    def build():
        bl.clear()
        bl.bulk_build(allk, allv, allo)
    t_b = timed(build)
    ob = _sub_oracle(B)
    ob.bulk_build(np.concatenate([x[0] for x in sub]), np.concatenate([x[1] for x in sub]),
                  np.concatenate([x[2] for x in sub]))
    rates, outs = _queries(bl, dev, dq, dk1, dk2, timed)
    fails, _ = check_queries(ob, PARITY_LO, PARITY_HI, q, outs[0], outs[1], k1, k2, *outs[2:])
    gate("N1 bulk build", fails)
    out["bulk_build"] = {"n": int(allk.numel()), "ms": t_b,
                         "melem_per_s": allk.numel() / (t_b * 1e-3) / 1e6, "r": bl.r,
                         "paper_K40c_melem_per_s": "770 (KV sort) / 728 (bulk build), PAPER.md:860"}
    bl.close()
    del allk, allv, allo
    out["workload"] = ("C3 batches: LSM and GPU SA at r=63 (2^24 queries, L=8), cleanup of the "
                       "6-level LSM; bulk build of all 64 batches")
    out["parity"] = "O1 on the key sub-range at r=63, after cleanup, and for the bulk build"
    return out


def extra_c4(pkg, dev, stream):
    """C4 (BASELINE configs[3]): b = 2^20 insert-only, r =
    127 (seven levels, n = 127*2^20) and r = 128 (one level, 2^27): count and
    range at L in {8, 128, 1024}, nq = min(2^24, 2^27 / L) (R16)."""
    import torch
    from paper_1707_05354_b200 import to_device
    timed = _ev_timer(stream)
    seed = synth.SEED_BASE + 3
    lsm = pkg.GpuLSM(B, reserve_batches=128)
    o1 = _sub_oracle(B)
    rows = []
    r = 0
    for target in (127, 128):
        while r < target:
            k, v, d = synth.updates(seed, r * B, B, delete_frac4=0)
            lsm.update(to_device(k, dev), to_device(v, dev), to_device(d, dev))
            m = (k >= PARITY_LO) & (k < PARITY_HI)
            o1.apply_batch(k[m], v[m], d[m])
            r += 1
        torch.cuda.synchronize()
        n = r * B
        for L in (8, 128, 1024):
            nq = min(1 << 24, (1 << 27) // L)
            k1, k2 = synth.range_queries(seed + L, nq, n, L)
            dk1, dk2 = to_device(k1, dev), to_device(k2, dev)
            cnt = torch.empty(nq, dtype=torch.int32, device=dev)
            t_c = timed(lambda: lsm.count_into(dk1, dk2, cnt))
            total = int(cnt.to(torch.int64).sum().item())
            roff = torch.empty(nq + 1, dtype=torch.int64, device=dev)
            rk = torch.empty(total + 16, dtype=torch.int32, device=dev)
            rv = torch.empty(total + 16, dtype=torch.int32, device=dev)
            got = []
            t_r = timed(lambda: got.append(lsm.range_into(dk1, dk2, roff, rk, rv)))
            fails, nchk = check_queries(o1, PARITY_LO, PARITY_HI, None, None, None, k1, k2, cnt,
                                        roff, rk, rv)
            gate(f"C4 r={r} L={L}", fails + ([] if got[-1] == total else ["count != len(range)"]))
            rows.append({"r": r, "levels": bin(r).count("1"), "L": L, "nq": nq,
                         "count_mqps": nq / (t_c * 1e-3) / 1e6, "range_mqps": nq / (t_r * 1e-3) / 1e6,
                         "pairs_per_query": total / nq,
                         "range_out_GBps": total * 8 / (t_r * 1e-3) / 1e9,
                         "checked_ranges": nchk.get("ranges")})
            del rk, rv, roff, cnt
    lsm.close()
    return {"workload": "C4: b=2^20 insert-only, r in {127 (7 levels), 128 (1 level)}, "
                        "L in {8, 128, 1024}, nq = min(2^24, 2^27/L)",
            "rows": rows, "parity": "O1 on the key sub-range; count == len(range) on every row",
            "full_sweep": "scripts/sweep_c4.py (r in 96..128, L in 8..1024)"}


def run_reference(args):
    """--impl reference: the CPU oracle on this arm's config (bounded samples)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    seed = synth.SEED_BASE + 2
    per_step = 2  # batches of 2^20 per step (bounded sample)
    data = [synth.updates(seed, j * B, B, delete_frac4=1) for j in range(per_step)]
    threads = os.cpu_count() or 1
    times = []
    for it in range(args.warmup + args.steps):
        o = oracle.ShardedOracleDict(B, threads)
        t0 = time.perf_counter()
        for k, v, d in data:
            o.apply_batch(k, v, d)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = args.steps * per_step * B / tot / 1e6
    sample = (f"{per_step} C3 batches (2x2^20 mixed updates) per step into fresh std::maps, "
              f"{threads} key-range shards, one thread each")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "b": B, "batches": R},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


C5_B = 1 << 24
C5_NQ = 1 << 26
C5_LO, C5_HI = 5 << 22, 6 << 22  # parity sub-range: 1/512 of the key domain


def run_c5_single(args):
    """--config c5 at N = 1 (BASELINE configs[4] on one GPU): global batch
    b = 2^24 mixed 75/25, 64 batches from empty -> 2^30 resident records,
    then 2^26 lookups (50 % hit). A batch of 2^24 takes the multi-wave
    onesweep LSD sort. Inputs are generated in device memory
    (synth's torch copy of the generator); lookups inside the key sub-range
    [5*2^22, 6*2^22) are checked against O1 fed the updates in that range."""
    import torch
    import oracle
    import paper_1707_05354_b200 as pkg
    from paper_1707_05354_b200 import to_numpy_u32
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    seed = synth.SEED_BASE + 4
    t0 = time.time()
    batches = [synth.updates_t(seed, j * C5_B, C5_B, delete_frac4=1, device=dev) for j in range(R)]
    q = synth.lookup_queries_t(seed, C5_NQ, R * C5_B, device=dev)
    gen_s = time.time() - t0
    lsm = pkg.GpuLSM(C5_B, reserve_batches=R)
    stream = torch.cuda.current_stream()
    lv = torch.empty(C5_NQ, dtype=torch.int32, device=dev)
    lf = torch.empty(C5_NQ, dtype=torch.uint8, device=dev)

    def step(rec):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        lsm.clear()
        e[0].record(stream)
        for k, v, d in batches:
            lsm.update(k, v, d)
        e[1].record(stream)
        lsm.lookup_into(q, lv, lf)
        e[2].record(stream)
        if rec is not None:
            rec.append(e)

    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize()
    recs = []
    l0 = lsm.launch_count
    with ClockSampler(0) as clk:
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for _ in range(args.steps):
            step(recs)
        stop.record(stream)
        torch.cuda.synchronize()
    launches = lsm.launch_count - l0
    upd = float(np.mean([e[0].elapsed_time(e[1]) for e in recs]))
    look = float(np.mean([e[1].elapsed_time(e[2]) for e in recs]))
    lsm.profile_enable(True)
    step(None)
    torch.cuda.synchronize()
    prof = lsm.profile_read()
    lsm.profile_enable(False)
    # parity: lookups inside the sub-range vs O1 fed the sub-range updates
    o1 = oracle.OracleDict(C5_B)
    for k, v, d in batches:
        m = (k >= C5_LO) & (k < C5_HI)  # keys < 2^31: int32 compares are exact
        o1.apply_batch(to_numpy_u32(k[m]), to_numpy_u32(v[m]), d[m].cpu().numpy())
    qh = to_numpy_u32(q)
    fails, nchk = check_queries(o1, C5_LO, C5_HI, qh, lv, lf)
    gate("C5 (N=1)", fails)
    peak, peak_src = measured_peaks()
    per_class = {c: {"ms_per_step": p["ms"], "launches_per_step": p["launches"],
                     "alg_GBps": (p["alg_bytes"] / (p["ms"] * 1e-3) / 1e9) if p["ms"] else None}
                 for c, p in prof.items() if p["launches"]}
    dom = max(prof, key=lambda c: prof[c]["ms"])
    ach = prof[dom]["alg_bytes"] / (prof[dom]["ms"] * 1e-3) / 1e9
    line = {"metric": METRIC, "value": R * C5_B / (upd * 1e-3) / 1e6, "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": start.elapsed_time(stop) / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (splitmix64 uniform 31-bit keys, generated on the device)",
            "config": {"workload": "C5 on one GPU: b=2^24 mixed 75/25, 64 batches -> 2^30 resident; "
                                   "2^26 lookups (50% hit)", "b": C5_B, "batches": R,
                       "resident": R * C5_B, "nq": C5_NQ, "parallelism": "1 GPU"},
            "update_ms_per_step": upd, "lookup_mqps": C5_NQ / (look * 1e-3) / 1e6,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": ach / peak,
                         "traffic": None},
            "kernels": per_class, "gpu_launches": launches, "clocks": clk.summary(),
            "parity": {"ok": True, **nchk, "oracle": "O1 on the key sub-range [5*2^22, 6*2^22)"},
            "input_gen_s": gen_s}
    print(json.dumps(line), flush=True)
    return 0


def run_native(args):
    import torch
    import paper_1707_05354_b200 as pkg
    from paper_1707_05354_b200 import to_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1 or args.sharded:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local_rank))
        from paper_1707_05354_b200.sharded import run_sharded_bench
        return run_sharded_bench(args, dist, rank, world, local_rank, clock_cls=ClockSampler,
                                 peaks_fn=measured_peaks)

    seed = synth.SEED_BASE + 2
    dev = torch.device("cuda", local_rank)
    # ---- inputs resident in HBM before timing ----
    t0 = time.time()
    keys_d, vals_d, ops_d = [], [], []
    host_batches = []
    sub = []  # the updates inside the parity sub-range (oracle input)
    for j in range(R):
        k, v, d = synth.updates(seed, j * B, B, delete_frac4=1)
        m = (k >= PARITY_LO) & (k < PARITY_HI)
        sub.append((k[m], v[m], d[m]))
        keys_d.append(to_device(k, dev))
        vals_d.append(to_device(v, dev))
        ops_d.append(to_device(d, dev))
        if args.e2e:
            host_batches.append((torch.from_numpy(k.view(np.int32)).pin_memory(),
                                 torch.from_numpy(v.view(np.int32)).pin_memory(),
                                 torch.from_numpy(d).pin_memory()))
    n_res = R * B
    q_host = synth.lookup_queries(seed, NQ, n_res)
    q_look = to_device(q_host, dev)
    k1, k2 = synth.range_queries(seed, NQ, n_res, L_RANGE)
    k1_d, k2_d = to_device(k1, dev), to_device(k2, dev)
    gen_s = time.time() - t0
    lv = torch.empty(NQ, dtype=torch.int32, device=dev)
    lf = torch.empty(NQ, dtype=torch.uint8, device=dev)
    cnt = torch.empty(NQ, dtype=torch.int32, device=dev)
    roff = torch.empty(NQ + 1, dtype=torch.int64, device=dev)
    rcap = 16 * NQ
    rk = torch.empty(rcap, dtype=torch.int32, device=dev)
    rv = torch.empty(rcap, dtype=torch.int32, device=dev)

    lsm = pkg.GpuLSM(B, reserve_batches=R)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    levels_searched = [1, 1]

    def step(record):
        e = [ev() for _ in range(10)]
        lsm.clear()
        e[0].record(stream)
        for j in range(R):
            lsm.update(keys_d[j], vals_d[j], ops_d[j])
        e[1].record(stream)
        lsm.lookup_into(q_look, lv, lf)
        e[2].record(stream)
        lsm.count_into(k1_d, k2_d, cnt)
        e[3].record(stream)
        tot_pre = lsm.range_into(k1_d, k2_d, roff, rk, rv)
        e[4].record(stream)
        levels_searched[0] = lsm.query_levels
        lsm.cleanup()
        e[5].record(stream)
        levels_searched[1] = lsm.query_levels
        lsm.lookup_into(q_look, lv, lf)
        e[6].record(stream)
        lsm.count_into(k1_d, k2_d, cnt)
        e[7].record(stream)
        tot_post = lsm.range_into(k1_d, k2_d, roff, rk, rv)
        e[8].record(stream)
        if record is not None:
            record.append((e, tot_pre, tot_post))

    # warm-up
    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize()
    levels_before = bin(R).count("1")
    recs = []
    l0 = lsm.launch_count
    # timed region: no per-launch events (they would split every launch pair
    # and defeat programmatic dependent launch); CUDA events per phase only
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        start, stop = ev(), ev()
        start.record(stream)
        for _ in range(args.steps):
            step(recs)
        stop.record(stream)
        torch.cuda.synchronize()
    launches = lsm.launch_count - l0
    # per-kernel-class breakdown for the roofline: the same K steps again with
    # the library's per-launch CUDA events on the launching stream
    lsm.profile_enable(True)
    for _ in range(args.steps):
        step(None)
    torch.cuda.synchronize()
    prof = lsm.profile_read()
    lsm.profile_enable(False)
    # SURVEY §8(d) byte model for the query classes (per query; levels = the
    # sorted runs searched, E[candidates] = L by the generator, R15):
    #   lookup 9 + 32*levels + 32*hit, count 12 + 64*levels + 4*L,
    #   range 20 + 64*levels + 12*L + 8*valid
    hit = float(lf.to(torch.float32).mean().item())
    lv_pre, lv_post = levels_searched
    pairs = recs[-1][1] + recs[-1][2]
    model = {
        # encode + sort: §8(d)'s 70 B/update (the onesweep-LSD figure; the
        # MSD + rank implementation moves 41 B of it)
        "sort_pass": 70.0 * R * B,
        "lookup": NQ * (2 * 9 + 32 * (lv_pre + lv_post) + 2 * 32 * hit),
        "count": NQ * (2 * 12 + 64 * (lv_pre + lv_post) + 2 * 4 * L_RANGE),
        "range": NQ * (2 * 20 + 64 * (lv_pre + lv_post) + 2 * 12 * L_RANGE) + 8 * pairs,
    }
    # cleanup (count + write + placebo fill; the merges are in "merge"):
    # read 8n, write 8r'b
    model["cleanup"] = 8.0 * R * B + 8.0 * lsm.r * B
    for c, bytes_per_step in model.items():
        if c in prof:
            prof[c]["alg_bytes"] = bytes_per_step * args.steps
    total_ms = start.elapsed_time(stop)
    # ---- parity gate: the last step's outputs vs O1 ----
    parity = parity_gate(lsm, sub, q_host, k1, k2, lv, lf, cnt, roff, rk, rv, recs[-1][1],
                         recs[-1][2])
    ph = np.zeros(8)
    for e, _, _ in recs:
        for i in range(8):
            ph[i] += e[i].elapsed_time(e[i + 1])
    ph /= args.steps
    r_after = lsm.r
    upd_ms = ph[0]
    value = R * B / (upd_ms * 1e-3) / 1e6

    # ---- roofline of the dominant kernel class ----
    peak, peak_src = measured_peaks()
    dom = max(prof, key=lambda c: prof[c]["ms"])
    ach = prof[dom]["alg_bytes"] / (prof[dom]["ms"] * 1e-3) / 1e9 if prof[dom]["ms"] else 0.0
    step_kernel_ms = sum(p["ms"] for p in prof.values())
    traffic, traffic_src = None, None
    summ = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(summ):
        with open(summ) as f:
            tr = json.load(f)
        if dom in tr:  # DRAM bytes of one captured launch of this kernel (ncu --set full)
            traffic = tr[dom].get("dram_bytes_per_launch")
            traffic_src = f"profiles/ncu_traffic.json ({tr[dom].get('kernel')}, {tr[dom].get('rep')})"
    alg_per_launch = prof[dom]["alg_bytes"] / max(prof[dom]["launches"], 1)
    # what the kernel's DRAM actually moved per launch (ncu) over its live
    # event time, and -- for the random-access classes -- the rate of random
    # 128-byte line fills against the ceiling measured by scripts/rand_probe.cu
    dram_live = None
    if traffic:
        t_live = prof[dom]["ms"] / max(prof[dom]["launches"], 1) * 1e-3
        dram_live = {"GBps": traffic / t_live / 1e9, "frac": traffic / t_live / 1e9 / peak}
        rp = os.path.join(ROOT, "profiles", "rand_probe.json")
        if dom in ("lookup", "count", "range") and os.path.exists(rp):
            with open(rp) as f:
                ceil = json.load(f)
            lines = traffic / ceil["bytes_per_random_read"] / t_live
            dram_live["random_lines_per_s"] = lines
            dram_live["random_line_ceiling_per_s"] = ceil["random_reads_per_s"]
            dram_live["frac_of_random_ceiling"] = lines / ceil["random_reads_per_s"]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak,
                "peak_source": peak_src, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "traffic_source": traffic_src,
                "alg_bytes_per_launch": alg_per_launch,
                "dram_live": dram_live,
                "timing": "per-launch CUDA events on the launching stream over K more identical "
                          "steps right after the timed ones (the timed steps run without them: "
                          "per-launch events split programmatic dependent launch)",
                "share_of_step_kernel_time": prof[dom]["ms"] / step_kernel_ms if step_kernel_ms else None,
                "byte_model": ("SURVEY §8(d) per-unit figures: sort 70 B/update (the MSD + rank "
                               "implementation moves 41 B), merge 16 B per output record, lookup "
                               "9+32*levels+32*hit, count 12+64*levels+4*L, range "
                               "20+64*levels+12*L+8*valid B/query (E[candidates]=L, R15), cleanup "
                               "8n + 8r'b"),
                "levels_searched": {"before_cleanup": levels_searched[0],
                                    "after_cleanup": levels_searched[1]}}
    per_class = {c: {"ms_per_step": p["ms"] / args.steps,
                     "launches_per_step": p["launches"] / args.steps,
                     "alg_GBps": (p["alg_bytes"] / (p["ms"] * 1e-3) / 1e9) if p["ms"] else None,
                     "frac_of_peak": ((p["alg_bytes"] / (p["ms"] * 1e-3) / 1e9) / peak) if p["ms"] else None}
                 for c, p in prof.items() if p["launches"]}
    queries = {
        "nq": NQ, "L": L_RANGE,
        "lookup_mqps_before_cleanup": NQ / (ph[1] * 1e-3) / 1e6,
        "count_mqps_before_cleanup": NQ / (ph[2] * 1e-3) / 1e6,
        "range_mqps_before_cleanup": NQ / (ph[3] * 1e-3) / 1e6,
        "lookup_mqps_after_cleanup": NQ / (ph[5] * 1e-3) / 1e6,
        "count_mqps_after_cleanup": NQ / (ph[6] * 1e-3) / 1e6,
        "range_mqps_after_cleanup": NQ / (ph[7] * 1e-3) / 1e6,
        "levels_before_cleanup": levels_before,
        "levels_after_cleanup": bin(r_after).count("1"),
        "range_pairs_before": recs[-1][1], "range_pairs_after": recs[-1][2],
    }
    cleanup = {"ms": ph[4], "melem_per_s": n_res / (ph[4] * 1e-3) / 1e6,
               "r_after": r_after}

    # ---- e2e: updates through the public API from pinned host buffers ----
    e2e = None
    if args.e2e:
        def e2e_step():
            lsm.clear()
            for (hk, hv, hd) in host_batches:
                lsm.update_host(hk, hv, hd)
            lsm.sync()  # D2H of the sticky status word: the step's result
        for _ in range(1):
            e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.steps
        e2e = {"value": R * B / dt / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": R * B * 9, "d2h_bytes_per_step": 4,
               "note": "lsm_update_host x64 (pinned H2D on the library's copy stream, double-"
                       "buffered so batch j+1's copy overlaps batch j's update) + lsm_sync, "
                       "wall clock"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic (splitmix64 uniform 31-bit keys)",
        "config": {"workload": WORKLOAD, "b": B, "batches": R, "resident": n_res,
                   "mix": "75% insert / 25% delete", "nq": NQ, "L": L_RANGE,
                   "l2": "inputs larger than L2 (600 MB updates, 512 MB levels) -- no flush"},
        "update_ms_per_step": upd_ms,
        "phase_ms": {"update": ph[0], "lookup": ph[1], "count": ph[2], "range": ph[3],
                     "cleanup": ph[4], "lookup_post": ph[5], "count_post": ph[6],
                     "range_post": ph[7]},
        "parity": parity,
        "queries": queries, "cleanup": cleanup,
        "roofline": roofline, "kernels": per_class,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
        "input_gen_s": gen_s,
    }
    if args.extra:
        t_x = time.time()
        sec = {}
        sec["c2"] = extra_c2(pkg, dev, stream)
        sec["c3_r63_sa_bulk"] = extra_c3p_sa_bulk(pkg, dev, stream, keys_d, vals_d, ops_d, sub,
                                                  q_host, k1, k2)
        sec["c4"] = extra_c4(pkg, dev, stream)
        sec["seconds"] = time.time() - t_x
        line["secondary"] = sec
    if args.cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_oracle()
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-extra", dest="extra", action="store_false",
                    help="skip the secondary configurations (C2, C3' + SA + bulk build, C4)")
    ap.add_argument("--config", default="c3", choices=["c3", "c5"],
                    help="c3 (default): BASELINE configs[2]; c5: configs[4] (global b = 2^24, "
                         "2^30 resident; strong scaling under torchrun)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the key-range sharded router even at N=1")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c5" and int(os.environ.get("WORLD_SIZE", "1")) == 1 and not args.sharded:
        return run_c5_single(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
