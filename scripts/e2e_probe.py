"""Repeats the bench's e2e measurement (pinned host buffers through qnb_plan_forward) to
show its run-to-run spread, next to the bare H2D copy of the same bytes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench


class A:
    model = "alexnet"; precision = "int8"; batch = 256; steps = 20; warmup = 5


wl = bench.Workload(A, 0, 1)
x_pin = torch.from_numpy(wl.x_host).pin_memory()
o_pin = torch.empty((256, 1000), dtype=torch.float32).pin_memory()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    wl.step_e2e(x_pin, o_pin)
torch.cuda.synchronize()
for rep in range(6):
    e0.record(st)
    for _ in range(20):
        wl.step_e2e(x_pin, o_pin)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    h = torch.empty_like(wl.x_dev)
    e0.record(st)
    for _ in range(20):
        h.copy_(x_pin, non_blocking=True)
    e1.record(st)
    torch.cuda.synchronize()
    hm = e0.elapsed_time(e1) / 20
    print(f"rep {rep}: e2e {ms:.3f} ms/step = {256 / ms * 1e3:.0f} img/s   h2d {hm:.3f} ms", flush=True)
