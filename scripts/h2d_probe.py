"""Pinned host -> device copy bandwidth on this box (the e2e path's bound):
one stream with 1/4/9/64 MB copies, and three arrays per batch as the
library's staging does (keys 4 B, values 4 B, ops 1 B per update)."""
import time
import torch

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
for mb in (1, 4, 9, 64, 256):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    reps = max(4, 2048 // mb)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"H2D {mb:4d} MB x {reps}: {reps * n / (ms * 1e-3) / 1e9:.1f} GB/s", flush=True)
b = 1 << 20
hk = torch.empty(b, dtype=torch.int32).pin_memory()
hv = torch.empty(b, dtype=torch.int32).pin_memory()
ho = torch.empty(b, dtype=torch.uint8).pin_memory()
dk = torch.empty(b, dtype=torch.int32, device=dev)
dv = torch.empty(b, dtype=torch.int32, device=dev)
do = torch.empty(b, dtype=torch.uint8, device=dev)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
with torch.cuda.stream(s):
    for _ in range(256):
        dk.copy_(hk, non_blocking=True)
        dv.copy_(hv, non_blocking=True)
        do.copy_(ho, non_blocking=True)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"batch of 2^20 updates as 3 arrays (9 MB): {256 * 9 * b / (ms * 1e-3) / 1e9:.1f} GB/s, "
      f"{256 * b / (ms * 1e-3) / 1e6:.0f} M updates/s", flush=True)
