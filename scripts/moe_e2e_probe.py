import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from types import SimpleNamespace
a = SimpleNamespace(model="alexnet_moe", precision="int8", batch=256)
wl = bench.Workload(a, 0, 1)
x_pin = torch.from_numpy(wl.x_host).pin_memory()
o_pin = torch.empty((256, 1000), dtype=torch.float32).pin_memory()
res = {}
for mode in ["dev", "e2e", "dev", "e2e"]:
    ts = []
    for _ in range(6):
        torch.cuda.synchronize(); t = time.perf_counter()
        if mode == "dev": wl.step()
        else: wl.step_e2e(x_pin, o_pin)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
    print(mode, [round(x, 2) for x in ts], flush=True)
