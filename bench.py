#!/usr/bin/env python
"""AlexNet INT8 batch-256 inference on B200 through the compiled qnb plan
(BASELINE.json metric: AlexNet INT8/FP16 images/sec at 1/2/4/8 B200; conv TOPS vs
int8 tensor peak).

    python bench.py [--gpus N --steps K --warmup W]            # this framework
    python bench.py --impl reference [--steps K --warmup W]     # the reference's CPU path
    torchrun --nproc-per-node N bench.py --gpus N ...          # weak scaling, 256 img/GPU

A step is one forward of one batch of synthetic 227x227 images (seeded U(0,255)),
seeded random-init weights, calibration fixture tests/golden/alexnet_int8_calib.json.
The input batch (158 MB FP32) is larger than the 126 MB L2, so no explicit flush is
needed between steps.  One JSON line is printed by rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "AlexNet INT8 images/sec (batch 256 per GPU, 227x227)"
METRICS = {
    "alexnet": "AlexNet {P} images/sec (batch {B} per GPU, 227x227)",
    "alexnet_moe": "AlexNet-MoE {P} images/sec (16 experts top-4, batch {B} per GPU, 227x227)",
    "vgg16": "VGG-16 {P} images/sec (batch {B} per GPU, 224x224)",
}
CONFIG_IDX = {"alexnet": 1, "alexnet_moe": 2, "vgg16": 3}


def metric_name(model, precision, batch):
    return METRICS.get(model, "{M} {P} images/sec (batch {B})").format(M=model, P=precision.upper(), B=batch)
DT = {"fp32": 0, "fp16": 1, "int8": 2, "int16": 3}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="qnb", choices=["qnb", "reference"])
    ap.add_argument("--model", default="alexnet")
    ap.add_argument("--precision", default="int8")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--cpu-threads", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-reps", type=int, default=3)
    ap.add_argument("--sweep-ck", default="", help="convsweep: comma list of C=K values (default 64,128,256,512)")
    return ap.parse_args()


# ------------------------------------------------------------------ distributed
def dist_setup(use_cuda: bool):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if use_cuda else "gloo")
    return ws, rank, local


def barrier(ws, device=None):
    if ws > 1:
        import torch.distributed as dist
        if device is not None:
            dist.barrier(device_ids=[device])
        else:
            dist.barrier()


def max_over_ranks(x: float, ws: int, device=None) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks and throttle reasons."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop_flag = [], set(), False
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop_flag:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_flag = True
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ model setup
def model_setup(model: str, precision: str):
    from paper_2209_15427_b200 import graph as G
    from paper_2209_15427_b200 import graphs
    g = graphs.MODELS[model](1)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    if any(l["kind"] == "moe" for l in g["layers"]):
        params = graphs.synth_params_moe(g)
    else:
        params = graphs.synth_params(g, shapes)
    # OBSERVE ranges are FP32 statistics, independent of the target precision: every
    # precision finalizes its grids from the same calibration fixture
    path = os.path.join(ROOT, "tests", "golden", f"{model}_{precision}_calib.json")
    if not os.path.exists(path):
        path = os.path.join(ROOT, "tests", "golden", f"{model}_int8_calib.json")
    with open(path) as f:
        ranges = json.load(f)["ranges"]
    return g, shapes, params, ranges


def reference_nets(g, precision, params, ranges, n):
    """n independent reference Nets (one per host thread), built in parallel."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import ffi
    ref = ffi.Reference()

    def one(_):
        net = ref.net(json.dumps(g), DT[precision])
        for k, v in params.items():
            net.set_param(k, v)
        for k, (lo, hi) in ranges.items():
            net.set_range(k, lo, hi)
        net.finalize()
        net.set_mode(3 if precision in ("int8", "int16") else 0)
        return net

    with ThreadPoolExecutor(max_workers=min(n, 16)) as ex:
        return list(ex.map(one, range(n)))


def cpu_forward_rate(nets, x, out_bytes):
    from oracle import ffi
    t0 = time.perf_counter()
    ffi.forward_mt(nets, "data", x, "prob", out_bytes)
    return x.shape[0] / (time.perf_counter() - t0)


# ------------------------------------------------------------------ arms
def run_reference(a):
    ws, rank, local = dist_setup(use_cuda=False)
    if rank != 0:
        return
    from oracle import ffi
    if not ffi.have_reference():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return
    g, shapes, params, ranges = model_setup(a.model, a.precision)
    T = os.cpu_count() or 1
    T = min(T, 64)
    nets = reference_nets(g, a.precision, params, ranges, T)
    from paper_2209_15427_b200 import graphs
    x = graphs.synth_images(T, shapes["data"][1:], offset=0)
    for _ in range(a.warmup):
        cpu_forward_rate(nets, x, 4000)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        cpu_forward_rate(nets, x, 4000)
    dt = time.perf_counter() - t0
    v = T * a.steps / dt
    line = {"impl": "reference", "metric": metric_name(a.model, a.precision, a.batch), "value": v, "unit": "images/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt / a.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic U(0,255) images, seeded random-init weights",
            "config": {"workload": f"{a.model} {a.precision} forward, bounded sample of {T} images "
                                   f"per step (reference Net::forward, QUANTIZED mode)", "global_batch": T,
                       "parallelism": f"{T} host threads, one Net each"},
            "cpu_baseline": {"value": v, "unit": "images/s", "cores": T, "kind": "reference",
                             "sample": f"{T} images per step x {a.steps} steps"},
            "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


class Workload:
    """The measured hot path for one rank: a compiled plan (chain nets) or the MoE
    executor, with device input/output buffers and a step() that runs one forward."""

    def __init__(self, a, rank, ws):
        import torch
        from paper_2209_15427_b200 import graph as G
        from paper_2209_15427_b200 import graphs
        from paper_2209_15427_b200.net import QUANTIZED, Net
        g, shapes, params, ranges = model_setup(a.model, a.precision)
        self.g, self.shapes, self.params, self.ranges = g, shapes, params, ranges
        self.moe = any(l["kind"] == "moe" for l in g["layers"])
        gg = G.override_precision(g, a.precision) if a.precision != "fp32" else g
        if self.moe:
            from paper_2209_15427_b200.moe import MoeNet
            net = MoeNet(gg, rank=rank, world=ws)
        else:
            net = Net(gg)
        for k, v in params.items():
            net.set_param(k, v)
        for k, (lo, hi) in ranges.items():
            net.set_range(k, lo, hi)
        net.finalize_quantizers()
        net.set_quant_mode(QUANTIZED)
        self.net = net
        B = self.B = a.batch
        self.x_host = graphs.synth_images(B, shapes["data"][1:], offset=rank * B)
        self.x_dev = torch.from_numpy(self.x_host).cuda()
        self.n_out = 1000
        self.out_dev = torch.empty((B, self.n_out), dtype=torch.float32, device="cuda")
        self.sp = torch.cuda.current_stream().cuda_stream
        if self.moe:
            self.plan = None
            self.kernels = net.moe_plan(B).kernels_per_forward() if ws == 1 else None
        else:
            self.plan = net.compile(B)
            self.kernels = self.plan.stats()["kernels_per_forward"]

    def step(self):
        if self.moe:
            self.net.forward_device(self.x_dev.data_ptr(), self.out_dev.data_ptr(), self.B)
        else:
            self.plan.forward_device(self.x_dev.data_ptr(), self.out_dev.data_ptr(), self.B, self.sp)

    def step_e2e(self, x_pin, o_pin):
        if self.moe:  # host buffers: the trunk plan pipelines the H2D copy under its compute
            self.net.forward_device(x_pin.data_ptr(), o_pin.data_ptr(), self.B, in_host=True, out_host=True)
        else:
            self.plan.forward_device(x_pin.data_ptr(), o_pin.data_ptr(), self.B, self.sp, in_host=True,
                                     out_host=True)


def parity_check(wl, a, ref_prob, T):
    """The bench's own batch against the reference on the cpu_baseline sample: the GPU
    rows 0..T-1 of the timed batch-B forward vs reference Net::forward on the same images
    (prob: FP32 sink, ulp distance; for chain nets also the last quantized blob before the
    softmax, read from the plan and compared bit for bit with a reference prefix net)."""
    out = wl.out_dev[:T].cpu().numpy()
    ulp = np.abs(out.view(np.int32).astype(np.int64) - ref_prob.view(np.int32).astype(np.int64))
    res = {"images": T, "rows": f"0..{T - 1} of the timed batch of {wl.B}", "prob_max_ulp": int(ulp.max()),
           "prob_rows_bit_identical": int((ulp.max(axis=1) == 0).sum())}
    if a.precision in ("fp16", "fp32"):
        # north_star tolerance for float graphs: max-abs <= 1e-2 x the activation range
        d = float(np.abs(out.astype(np.float64) - ref_prob.astype(np.float64)).max())
        rng = float(ref_prob.max() - ref_prob.min())
        res.update({"prob_max_abs": d, "prob_range": rng, "within_1e-2_of_range": d <= 1e-2 * rng})
    top1 = (out.argmax(axis=1) == ref_prob.argmax(axis=1)).sum()
    res["top1_agree"] = int(top1)
    if wl.plan is None or a.precision not in ("int8", "int16"):
        return res
    from oracle import ffi
    from paper_2209_15427_b200 import graph as G
    layers = wl.g["layers"]
    names = [l["name"] for l in layers]
    ck = names[-2]  # the layer feeding the softmax (fc8)
    prefix = {"name": "prefix", "layers": layers[: names.index(ck) + 1]}
    pp = {k: v for k, v in wl.params.items() if k.split(".")[0] in names[: names.index(ck) + 1]}
    per = int(np.prod(G.infer_blobs(prefix)[ck]["shape"][1:]))
    es = 1 if a.precision == "int8" else 2
    nets = reference_nets(prefix, a.precision, pp, wl.ranges, T)
    theirs = ffi.forward_mt(nets, "data", wl.x_host[:T], ck, per * es).view(np.uint8 if es == 1 else np.uint16)
    raw, lay = wl.plan.blob(ck)
    n, h, w, cp, hh, hw, wx, e = lay
    mine = raw.view(theirs.dtype).reshape(n, h + 2 * hh, w + 2 * hw + wx, cp)[:T, hh, hw, :per]
    res.update({"int8_checkpoint": ck, "checkpoint_values": int(theirs.size),
                "checkpoint_mismatches": int((mine.reshape(-1) != theirs.reshape(T, per).reshape(-1)).sum())})
    return res


SWEEP_CK = (64, 128, 256, 512)
SWEEP_R = (3, 5, 11)
SWEEP_S = (1, 2, 4)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def int8_peak_tops(peaks):
    """Dense int8 tensor peak: the measured kind::i8 figure when the box has one
    (profiles/int8_peak.json, scripts/int8_peak.py), else 2 x the measured bf16 peak."""
    try:
        with open(os.path.join(ROOT, "profiles", "int8_peak.json")) as f:
            m = json.load(f)
        return float(m["int8_tops"]), f"measured kind::i8 ({m.get('how', 'profiles/int8_peak.json')})"
    except Exception:
        return 2.0 * peaks["bf16_tflops"], f"2 x bf16_tflops {peaks['bf16_tflops']} (dense int8 = 2x bf16)"


def fp16_peak_tflops(peaks):
    """Dense fp16 tensor peak: the measured kind::f16 MMA ceiling (profiles/int8_peak.json)
    when present, else the measured cuBLAS bf16 number (dense fp16 = bf16 on B200)."""
    try:
        with open(os.path.join(ROOT, "profiles", "int8_peak.json")) as f:
            m = json.load(f)
        return float(m["fp16_tflops"]), "measured kind::f16 MMA ceiling (profiles/int8_peak.json)"
    except Exception:
        return peaks["bf16_tflops"], "MEASURED_PEAKS.json bf16_tflops (dense fp16 = bf16)"


def run_convsweep(a):
    """BASELINE configs[4]: one convolution, N=128 (a.batch), 56x56, C=K in {64..512},
    R in {3, 5, 11} (pad R//2), stride in {1, 2, 4}, INT8 vs FP16.  Each shape is a
    compiled two-step plan (input pack + the conv); the conv kernel is timed with CUDA
    events on the plan's stream (plan.profile), after warm-up, inputs (> L2 for C >= 128)
    resident in HBM."""
    import torch
    from paper_2209_15427_b200 import graph as G
    from paper_2209_15427_b200 import graphs
    from paper_2209_15427_b200._lib import QnbError, check, lib
    from paper_2209_15427_b200.net import QUANTIZED, Net
    check(lib().qnb_device_check(0))
    peaks, src = load_peaks()
    i8_peak, i8_src = int8_peak_tops(peaks)
    f16_peak, f16_src = fp16_peak_tflops(peaks)
    N, res = a.batch if a.batch != 256 else 128, 56
    cks = [int(v) for v in a.sweep_ck.split(",")] if a.sweep_ck else SWEEP_CK
    rows = []
    tot = {"int8": [0.0, 0.0], "fp16": [0.0, 0.0]}
    launches0 = lib().qnb_kernel_launch_count()
    with ClockSampler(0) as clk:
        for C in cks:
            x = (torch.rand((N, C, res, res), device="cuda") * 255.0).contiguous()
            for R in SWEEP_R:
                for st in SWEEP_S:
                    g = graphs.conv_layer(N, C, res, C, R, st)
                    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
                    params = graphs.synth_params(g, shapes)
                    oh = shapes["conv"][2]
                    ops_ = 2.0 * N * oh * oh * C * C * R * R
                    row = {"C": C, "K": C, "R": R, "stride": st, "pad": R // 2, "out": oh, "gop": ops_ / 1e9}
                    for prec in ("int8", "fp16"):
                        net = Net(G.override_precision(g, prec))
                        for k, v in params.items():
                            net.set_param(k, v)
                        net.set_range("data", 0.0, 255.0)
                        net.set_range("conv", -150.0, 150.0)
                        net.finalize_quantizers()
                        net.set_quant_mode(QUANTIZED)
                        try:
                            plan = net.compile(N, use_cuda_graph=False)
                        except QnbError as e:
                            row[prec] = {"unsupported": str(e)[:120]}
                            continue
                        out = torch.empty(N * int(np.prod(plan.out_shape[1:])) * 4, dtype=torch.uint8,
                                          device="cuda")
                        plan.profile(x.data_ptr(), out.data_ptr(), N, 2, 0)  # warm-up
                        ms = plan.profile(x.data_ptr(), out.data_ptr(), N, a.profile_reps, 0)
                        steps = plan.steps()
                        j = next(i for i, s_ in enumerate(steps) if s_[1] == "igemm")
                        t = ms[j]
                        pk = i8_peak if prec == "int8" else f16_peak
                        tops = ops_ / (t * 1e-3) / 1e12
                        row[prec] = {"ms": round(t, 4), "tops": round(tops, 1), "frac": round(tops / pk, 3)}
                        tot[prec][0] += ops_
                        tot[prec][1] += t
                        del plan, net, out
                    rows.append(row)
                    print(json.dumps(row), file=sys.stderr, flush=True)
            del x
            torch.cuda.empty_cache()
    launches = lib().qnb_kernel_launch_count() - launches0
    agg = {p: (v[0] / (v[1] * 1e-3) / 1e12 if v[1] else None) for p, v in tot.items()}
    line = {"metric": "conv TOPS vs int8 tensor peak (single conv-layer sweep, BASELINE configs[4])",
            "value": agg["int8"], "unit": "TOPS", "n_gpus": 1, "steps": a.profile_reps, "warmup": 2,
            "ms_per_step": tot["int8"][1], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8 (s32 accumulate); f16 (f32 accumulate) alongside", "data": "synthetic U(0,255) input, "
            "seeded random-init weights",
            "config": {"workload": f"single conv layer, N={N}, {res}x{res}, C=K in {list(cks)}, R in {list(SWEEP_R)} "
                                   f"(pad R//2), stride in {list(SWEEP_S)}, INT8 vs FP16",
                       "parallelism": "dp1 (single GPU)",
                       "l2": "conv inputs for C >= 128 exceed the 126 MB L2; each step is one launch per shape"},
            "roofline": {"bound": "tensor", "achieved": agg["int8"], "peak": i8_peak, "unit": "TFLOP/s",
                         "frac": (agg["int8"] / i8_peak) if agg["int8"] else None, "traffic": None,
                         "peak_source": i8_src, "kernel": "igemm (all sweep shapes, ops-weighted)"},
            "fp16": {"tops": agg["fp16"], "peak": f16_peak, "peak_source": f16_src,
                     "frac": (agg["fp16"] / f16_peak) if agg["fp16"] else None},
            "e2e": None, "gpu_launches": int(launches), "clocks": clk.summary(), "per_shape": rows}
    print(json.dumps(line))


def run_qnb(a):
    import torch
    ws, rank, local = dist_setup(use_cuda=True)
    torch.cuda.set_device(local)
    from paper_2209_15427_b200._lib import check, lib

    check(lib().qnb_device_check(local))
    wl = Workload(a, rank, ws)
    B = wl.B
    stream = torch.cuda.current_stream()
    # N > 1: every rank classifies its own batch shard; the final logits are gathered
    # over NCCL (the path's only data-path collective besides the MoE all-to-all).  Chain
    # nets run through the C-ABI group (qnb_group_forward: plan + in-place ncclAllGather).
    gathered = torch.empty((ws * B, wl.n_out), dtype=torch.float32, device="cuda") if ws > 1 else None
    group = None
    if ws > 1 and not wl.moe:
        from paper_2209_15427_b200.group import Group
        group = Group.from_torch(rank, ws, local)

    def step():
        if group is not None:
            group.forward(wl.plan, wl.x_dev.data_ptr(), B, gathered.data_ptr(), wl.n_out * 4, wl.sp)
            return
        wl.step()
        if ws > 1:
            import torch.distributed as dist
            dist.all_gather_into_tensor(gathered, wl.out_dev)

    for _ in range(max(a.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches0 = lib().qnb_kernel_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier(ws, local)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(ws, local)
    launches = lib().qnb_kernel_launch_count() - launches0
    ms = e0.elapsed_time(e1)
    ms_max = max_over_ranks(ms, ws, local)
    value = ws * B * a.steps / (ms_max / 1e3)

    # end to end through the C-ABI with pinned host buffers (H2D input + D2H result per step)
    x_pin = torch.from_numpy(wl.x_host).pin_memory()
    o_pin = torch.empty((B, wl.n_out), dtype=torch.float32).pin_memory()
    # warm-up: at least W steps and ~1 s of sustained PCIe traffic (the first ~25-45
    # host-buffer steps after a device-only phase run up to 20 % slower while the link
    # ramps up; scripts/e2e_probe.py)
    t_w = time.perf_counter()
    n_w = 0
    while n_w < max(a.warmup, 3) or time.perf_counter() - t_w < 1.0:
        wl.step_e2e(x_pin, o_pin)
        torch.cuda.synchronize()
        n_w += 1
    torch.cuda.synchronize()
    barrier(ws, local)
    e0.record(stream)
    for _ in range(a.steps):
        wl.step_e2e(x_pin, o_pin)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws, local)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), ws, local)
    e2e_value = ws * B * a.steps / (e2e_ms / 1e3)
    # the PCIe bound of that number: the same pinned H2D copy alone
    h2d = torch.empty_like(wl.x_dev)
    e0.record(stream)
    for _ in range(a.steps):
        h2d.copy_(x_pin, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    h2d_ms = e0.elapsed_time(e1) / a.steps

    peaks, peak_src = load_peaks()
    int8_peak, int8_src = int8_peak_tops(peaks)
    # FP16 / FP32 graphs run kind::f16 / kind::tf32: their contractions are reported
    # against the measured dense fp16 (= bf16) peak
    f16_peak, f16_src = fp16_peak_tflops(peaks)
    mma_peak = int8_peak if a.precision in ("int8", "int16") else f16_peak
    hbm_peak = peaks["hbm_gbs"]
    per_layer, roof, conv_tops = [], None, None
    if wl.plan is not None:
        # per-step profile (events between steps, eager) -> roofline of the dominant kernel
        plan, net = wl.plan, wl.net
        ms_steps = plan.profile(wl.x_dev.data_ptr(), wl.out_dev.data_ptr(), B, a.profile_reps, wl.sp)
        steps_info = plan.steps()
        names = [l["name"] for l in net.graph["layers"]]
        conv_ops = conv_ms = 0.0
        for (li, kind, ops_, by), t in zip(steps_info, ms_steps):
            per_layer.append({"layer": names[li] if 0 <= li < len(names) else str(li), "kernel": kind,
                              "ms": round(t, 4),
                              "tops": round(ops_ / (t * 1e-3) / 1e12, 1) if ops_ else None,
                              "gbs": round(by / (t * 1e-3) / 1e9, 1)})
            if kind in ("igemm", "conv_pool") and names[li].startswith("conv"):
                conv_ops += ops_
                conv_ms += t
        dom = int(np.argmax(ms_steps))
        li, kind, ops_, by = steps_info[dom]
        t = ms_steps[dom]
        if kind in ("igemm", "conv_pool"):  # conv_pool: conv + ReLU + max-pool fused (qnb_front.cu)
            roof = {"bound": "tensor", "achieved": ops_ / (t * 1e-3) / 1e12, "peak": mma_peak, "unit": "TFLOP/s",
                    "op_type": ("int8 tensor ops (2 per u8 x u8 MAC), i.e. TOPS" if a.precision in ("int8", "int16")
                                else f"{a.precision} flops (2 per MAC)"),
                    "kernel": f"{kind} {names[li]}", "algorithmic_ops": ops_, "launch_ms": t}
        else:
            roof = {"bound": "hbm", "achieved": by / (t * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "kernel": f"{kind} {names[li]}", "algorithmic_bytes": by, "launch_ms": t}
        roof["frac"] = roof["achieved"] / roof["peak"]
        # measured DRAM traffic of that launch (dram__bytes_read + write, one ncu --set full
        # capture of this workload, committed under profiles/ncu/)
        roof["traffic"] = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu", f"traffic_{a.model}_{a.precision}.json")) as f:
                tr = json.load(f)["per_launch"].get(names[li])
            if tr:
                roof["traffic"] = tr["dram_bytes"]
                roof["traffic_source"] = f"profiles/ncu/traffic_{a.model}_{a.precision}.json"
                alg = roof.get("algorithmic_bytes") or by
                roof["algorithmic_bytes"] = alg
        except Exception:
            pass
        roof["peak_source"] = ((int8_src if a.precision in ("int8", "int16") else f16_src)
                               if kind in ("igemm", "conv_pool") else f"{peak_src}: hbm_gbs")
        conv_tops = conv_ops / (conv_ms * 1e-3) / 1e12 if conv_ms else None

    cpu = parity = None
    if rank == 0 and ws == 1 and not a.no_cpu_baseline:
        try:
            from oracle import ffi
            if ffi.have_reference():
                T = min(a.cpu_threads, os.cpu_count() or 1)
                if wl.moe:
                    T = min(T, 4)  # the MoE reference evaluates all 16 experts per image
                nets = reference_nets(wl.g, a.precision, wl.params, wl.ranges, T)
                xs = wl.x_host[:T]
                t0 = time.perf_counter()
                ref_prob = ffi.forward_mt(nets, "data", xs, "prob", 4000).view(np.float32).reshape(T, 1000)
                v = T / (time.perf_counter() - t0)
                cpu = {"value": v, "unit": "images/s", "cores": T, "kind": "reference",
                       "sample": f"{T} images of the same batch, one reference Net::forward thread each"}
                del nets
                parity = parity_check(wl, a, ref_prob, T)
        except Exception as e:  # reported, never fatal
            cpu = cpu or {"value": None, "error": str(e)[:200]}
            parity = parity or {"error": str(e)[:200]}

    if rank == 0:
        res = wl.x_host.shape[-1]
        line = {"metric": metric_name(a.model, a.precision, B), "value": value, "unit": "images/s", "n_gpus": ws,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "u8 (s32 accumulate)" if a.precision in ("int8", "int16") else a.precision,
                "data": f"synthetic U(0,255) images, seeded random-init weights",
                "config": {"workload": f"{a.model} {a.precision} forward, batch {B} per GPU, {res}x{res} "
                                       f"(BASELINE configs[{CONFIG_IDX.get(a.model, '?')}])",
                           "model": a.model, "global_batch": B * ws,
                           "parallelism": (f"dp{ws}: batch shard per GPU, NCCL all-gather of the logits "
                                           f"(qnb_group_forward)"
                                           + (", expert-parallel all-to-all" if wl.moe else "")) if ws > 1
                           else "dp1 (single GPU)",
                           "l2": f"input batch {wl.x_host.nbytes / 1e6:.0f} MB "
                                 + ("> 126 MB L2 (no flush needed)" if wl.x_host.nbytes > 126e6
                                    else "<= L2: activations are rewritten every step")},
                "e2e": {"value": e2e_value, "unit": "images/s",
                        "h2d_bytes_per_step": int(wl.x_host.nbytes), "d2h_bytes_per_step": int(B * wl.n_out * 4),
                        "h2d_only_ms": h2d_ms, "pcie_bound_images_per_s": B / (h2d_ms / 1e3)},
                "gpu_launches": int(launches), "kernels_per_forward": wl.kernels,
                "roofline": roof, "conv_tops": conv_tops, "conv_frac_of_peak":
                    (conv_tops / mma_peak if conv_tops else None),
                "conv_frac_of_spec_peak": (conv_tops / (4500.0 if a.precision in ("int8", "int16") else 2250.0)
                                           if conv_tops else None),
                "cpu_baseline": cpu, "parity": parity, "clocks": clk.summary(), "per_layer": per_layer}
        if wl.moe:
            line["moe_expert_counts_last_step"] = [int(c) for c in wl.net.last_stats["counts"]] \
                if hasattr(wl.net, "last_stats") else None
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.model == "convsweep":
        run_convsweep(a)
    else:
        run_qnb(a)


if __name__ == "__main__":
    main()
