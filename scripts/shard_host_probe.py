"""Host-side timing of ShardedLSM.update phases at world size 1 (diagnostic)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import synth
from paper_1707_05354_b200 import to_device
from paper_1707_05354_b200.sharded import ShardedLSM
b = 1 << 20
ins = [tuple(to_device(x) for x in synth.updates(5, j * b, b, delete_frac4=1)) for j in range(64)]
sh = ShardedLSM(b, reserve_batches=66)
acc = {"a2a": 0.0, "insert": 0.0}
orig_a2a, orig_ins = sh._a2a, sh._local_insert
def wrap(name, f):
    def g(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); acc[name] += time.perf_counter() - t; return r
    return g
sh._a2a = wrap("a2a", orig_a2a); sh._local_insert = wrap("insert", orig_ins)
for it in range(3):
    sh.clear(); torch.cuda.synchronize()
    for k in acc: acc[k] = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for j in range(64):
        sh.update(*ins[j])
    sh.flush()
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    print(f"host {1e3*(t1-t0):.1f} ms device {e0.elapsed_time(e1):.1f} ms  " + " ".join(f"{k} {1e3*v:.1f}" for k, v in acc.items()))
dist.destroy_process_group()
