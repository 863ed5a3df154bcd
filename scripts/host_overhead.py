"""Host enqueue time vs device time of the C3 update phase (diagnostic)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_1707_05354_b200 as pkg
from paper_1707_05354_b200 import to_device
b, R = 1 << 20, 64
seed = synth.SEED_BASE + 2
ins = []
for j in range(R):
    k, v, d = synth.updates(seed, j * b, b, delete_frac4=1)
    ins.append((to_device(k), to_device(v), to_device(d)))
lsm = pkg.GpuLSM(b, reserve_batches=R)
for it in range(4):
    lsm.clear()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for j in range(R):
        lsm.update(*ins[j])
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"enqueue {1e3*(t1-t0):.2f} ms  device {e0.elapsed_time(e1):.2f} ms  wall {1e3*(t2-t0):.2f} ms")
# raw C call cost without python marshalling
import ctypes
lib = lsm._lib
args = [(ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(d.data_ptr())) for k, v, d in ins]
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for it in range(3):
    lsm.clear(); torch.cuda.synchronize()
    e0.record(); t0 = time.perf_counter()
    for j in range(R):
        lib.lsm_update(lsm.h, args[j][0], args[j][1], args[j][2], b, s)
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    print(f"raw C: enqueue {1e3*(t1-t0):.2f} ms  device {e0.elapsed_time(e1):.2f} ms")
