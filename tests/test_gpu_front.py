"""The fused conv + ReLU + max-pool front kernel (csrc/qnb_front.cu) against the UNMODIFIED
reference Net (oracle/_ref) beyond the AlexNet shapes the other tests cover:

* a generic geometry (64 channels -> 16 per TMEM lane quarter, 99x99 input -> 23x23 conv ->
  11x11 pool; the run-time pixel-stride / row-width path, not the AlexNet specialisation);
* a requant whose shift is below 32 (the multiplier's low-word form of the fast requant):
  conv1's output grid made ~3x finer than its accumulator grid.

Reference semantics: conv_forward + relu_quant + pool_max (src/ops.cpp:264-342, 156-181,
344-390); the pool keeps its input's integer values (src/net.cpp:449-453)."""
import json

import numpy as np
import pytest

from oracle import ffi
from paper_2209_15427_b200 import graph as G
from paper_2209_15427_b200 import graphs
from paper_2209_15427_b200.graphs import _conv, _input, _ip, _pool, _relu, _softmax
from paper_2209_15427_b200.net import QUANTIZED, Net

pytestmark = pytest.mark.gpu
INT8 = 2


def ref_net(ref, g, params, ranges):
    net = ref.net(json.dumps(g), INT8)
    for k, v in params.items():
        net.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        net.set_range(k, lo, hi)
    net.finalize()
    net.set_mode(3)
    return net


def ours_net(g, params, ranges):
    net = Net(G.override_precision(g, "int8"))
    for k, v in params.items():
        net.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        net.set_range(k, lo, hi)
    net.finalize_quantizers()
    net.set_quant_mode(QUANTIZED)
    return net


def pool_blob(plan, name):
    raw, lay = plan.blob(name)
    n, h, w, cp, hh, hw, wx, es = lay
    return raw.view(np.uint8).reshape(n, h + 2 * hh, w + 2 * hw + wx, cp)[:, hh:hh + h, hw:hw + w, :]


def check_pool1(g, params, ranges, x):
    ref = ffi.Reference()
    ours = ours_net(g, params, ranges)
    out = ours.forward({"data": x})["prob"]
    plan = ours.plan(x.shape[0])
    assert "conv_pool" in [s[1] for s in plan.steps()]
    names = [l["name"] for l in g["layers"]]
    prefix = {"name": "prefix", "layers": g["layers"][: names.index("pool1") + 1]}
    pr = {k: v for k, v in params.items() if k.startswith("conv1.")}
    (arr, dt, qv), = ref_net(ref, prefix, pr, ranges).forward("data", x).values()
    mine = pool_blob(plan, "pool1")[..., : arr.shape[1]]
    theirs = np.transpose(arr, (0, 2, 3, 1))
    assert mine.shape == theirs.shape
    mism = int((mine != theirs).sum())
    assert mism == 0, f"pool1: {mism} of {theirs.size} differ"
    prob = ref_net(ref, g, params, ranges).forward("data", x)["prob"][0]
    d = np.abs(out.view(np.int32).astype(np.int64) - prob.view(np.int32).astype(np.int64))
    assert d.max() <= 1, d.max()


@pytest.mark.parametrize("batch", [5, 6])
def test_front_generic_geometry(batch):
    if not ffi.have_reference():
        pytest.skip("needs oracle/_ref")
    g = {"name": "front_generic", "layers": [
        _input("data", [1, 3, 99, 99]),
        _conv("conv1", "data", 64, 11, s=4), _relu("relu1", "conv1"), _pool("pool1", "relu1", 3, 2),
        _ip("fc", "pool1", 10), _softmax("prob", "fc"),
    ]}
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    params = graphs.synth_params(g, shapes, seed=7)
    ranges = {"data": (0.0, 255.0), "conv1": (-300.0, 310.0), "relu1": (0.0, 310.0), "fc": (-40.0, 45.0),
              "prob": (0.0, 1.0)}
    x = graphs.synth_images(batch, (3, 99, 99), offset=11)
    check_pool1(g, params, ranges, x)


def test_front_requant_shift_below_32():
    if not ffi.have_reference():
        pytest.skip("needs oracle/_ref")
    g = graphs.alexnet(1)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    params = graphs.synth_params(g, shapes)
    with open(__file__.replace("test_gpu_front.py", "golden/alexnet_int8_calib.json")) as f:
        ranges = {k: tuple(v) for k, v in json.load(f)["ranges"].items()}
    # conv1's output step ~1/3 of its accumulator step (scale_x * scale_w): the fixed-point
    # multiplier's shift lands below 32 (requant_from_ratio, src/quantizer.cpp:157-199)
    w = params["conv1.weight"]
    s_acc = (ranges["data"][1] - min(0.0, ranges["data"][0])) / 255.0 * (w.max() - min(0.0, w.min())) / 255.0
    half = 255.0 * s_acc / 3.0 / 2.0
    ranges["conv1"] = (-half, half)
    ranges["relu1"] = (0.0, half)
    x = graphs.synth_images(3, (3, 227, 227), offset=23)
    check_pool1(g, params, ranges, x)
