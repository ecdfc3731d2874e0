"""Per-step MoE forward times (device buffers), to characterise run-to-run variance."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench


class A:
    model = "alexnet_moe"; precision = "int8"; batch = 256; steps = 10; warmup = 3


wl = bench.Workload(A, 0, 1)
ts = []
for i in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    wl.step()
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print(" ".join(f"{t:.1f}" for t in ts))
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw,temperature.gpu", "--format=csv"], capture_output=True, text=True).stdout)
