"""Feasibility probe: do two independent C3 update streams overlap on one B200?
Handle A alone (64 batches of 2^20 on one stream) vs handles A and B fed
alternately on two streams. The aggregate rate tells how much of the update
phase is latency that a second, independent update sequence can fill.

    python scripts/overlap_handles.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1707_05354_b200 as pkg  # noqa: E402

b, nb = 1 << 20, 64
seed = synth.SEED_BASE + 2
torch.cuda.set_device(0)
K, V, D = synth.updates_t(seed, 0, nb * b, delete_frac4=1)
A = pkg.GpuLSM(b, reserve_batches=nb)
B = pkg.GpuLSM(b, reserve_batches=nb)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(handles, streams):
    for h, s in zip(handles, streams):
        h.clear(stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    s2.wait_event(e0)
    for j in range(nb):
        sl = slice(j * b, (j + 1) * b)
        for h, s in zip(handles, streams):
            h.update(K[sl], V[sl], D[sl], stream=s)
    for h, s in zip(handles, streams):
        h.sync(stream=s)  # joins the handle's merge stream (host wait)
    ej = torch.cuda.Event()
    ej.record(s2)
    s1.wait_event(ej)
    e1.record(s1)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for rep in range(3):
    t1 = run([A], [s1])
    t2 = run([A, B], [s1, s2])
    print(f"one handle: {t1:.3f} ms ({nb * b / t1 / 1e6:.1f} G/s); two handles on two streams: "
          f"{t2:.3f} ms ({2 * nb * b / t2 / 1e6:.1f} G/s aggregate)", flush=True)
