"""Host-timed breakdown of one AlexNet-MoE forward (synchronising after each stage)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from types import SimpleNamespace
a = SimpleNamespace(model="alexnet_moe", precision="int8", batch=256)
wl = bench.Workload(a, 0, 1)
net = wl.net
for _ in range(3):
    wl.step()
torch.cuda.synchronize()
import paper_2209_15427_b200.moe as M
orig = {}
times = {}
def wrap(obj, name, label):
    f = getattr(obj, name)
    def g(*args, **kw):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*args, **kw)
        torch.cuda.synchronize(); times[label] = times.get(label, 0) + time.perf_counter() - t
        return r
    setattr(obj, name, g)
p = net._pipe(256)
wrap(p["trunk"], "forward_device", "trunk")
wrap(p["gating"], "forward_device", "gating")
wrap(p["tail"], "forward_device", "tail")
for e, pl in p["experts"].items():
    wrap(pl, "forward_device", "experts")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    wl.step()
torch.cuda.synchronize(); tot = (time.perf_counter() - t0) / 5
print(json.dumps({"total_ms": tot * 1e3, **{k: v / 5 * 1e3 for k, v in times.items()},
                  "counts": [int(c) for c in net.last_stats["counts"]]}))
