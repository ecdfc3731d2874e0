"""Times the MoE e2e step's parts (H2D, forward, D2H) to explain the e2e number."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench


class A:
    model = "alexnet_moe"; precision = "int8"; batch = 256; steps = 10; warmup = 3


wl = bench.Workload(A, 0, 1)
x_pin = torch.from_numpy(wl.x_host).pin_memory()
o_pin = torch.empty((256, 1000), dtype=torch.float32).pin_memory()
for _ in range(3):
    wl.step()
torch.cuda.synchronize()
def timed(name, fn, n=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:12s} gpu {e0.elapsed_time(e1)/n:8.3f} ms  host {(time.perf_counter()-t0)*1e3/n:8.3f} ms", flush=True)
timed("forward", wl.step)
timed("h2d", lambda: wl.x_dev.copy_(x_pin, non_blocking=True))
timed("e2e", lambda: wl.step_e2e(x_pin, o_pin))
timed("forward", wl.step)
timed("e2e", lambda: wl.step_e2e(x_pin, o_pin), 20)
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    wl.step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
