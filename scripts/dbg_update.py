"""Debug: updates at several b with blocking launches; report the first failing call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1707_05354_b200 as pkg
from paper_1707_05354_b200 import to_device
for b in [int(x) for x in sys.argv[1:]] or [32768, 1 << 20]:
    g = pkg.GpuLSM(b)
    for j in range(6):
        k, v, d = synth.updates(1, j * b, b, delete_frac4=1)
        try:
            g.update(to_device(k), to_device(v), to_device(d))
            torch.cuda.synchronize()
        except Exception as e:
            print("b", b, "batch", j, "FAILED", e, flush=True)
            break
    else:
        print("b", b, "ok r=", g.r, flush=True)
