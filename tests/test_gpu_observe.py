"""OBSERVE-mode calibration on the device (Net::forward with QuantMode::OBSERVE,
src/net.cpp:305-330, observe() src/quantizer.cpp:58-68) against the ranges the
UNMODIFIED reference recorded over the same seeded images (tests/golden/*_calib.json,
made by tests/golden/make_calibration.py).  The device runs the float execution in
FP32 on TF32 tensor cores, so each recorded bound is compared within 1e-2 x the
blob's range magnitude (BASELINE.json north_star float tolerance)."""
import json
import os

import numpy as np
import pytest

from paper_2209_15427_b200 import graph as G
from paper_2209_15427_b200 import graphs
from paper_2209_15427_b200.net import OBSERVE, QUANTIZED, Net

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden(model):
    with open(os.path.join(HERE, "golden", f"{model}_int8_calib.json")) as f:
        return json.load(f)


def _net(model):
    g = graphs.MODELS[model](1)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    net = Net(G.override_precision(g, "int8"))
    for k, v in graphs.synth_params(g, shapes).items():
        net.set_param(k, v)
    return net, g, shapes


def test_observe_graph_is_float_execution():
    net, _, _ = _net("alexnet")
    og = net.observe_graph()
    kinds = [l["kind"] for l in og["layers"]]
    assert "quantizer" not in kinds
    assert all(l["top_data_type"] == G.FP32 and l["compute_data_type"] == G.FP32 for l in og["layers"])
    tops = {l["top"][0] for l in og["layers"]}
    for l in og["layers"]:
        for b in l.get("bottom", []):
            assert b in tops, b
    # every dropped quantizer top shares its bottom's calibration key
    for l in net.graph["layers"]:
        if l["kind"] == "quantizer":
            assert G.range_key(net.aliases, l["top"][0]) == G.range_key(net.aliases, l["bottom"][0])


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["lenet5", "vgg16_32", "alexnet"])
def test_observe_matches_reference_ranges(model):
    gold = _golden(model)
    net, g, shapes = _net(model)
    inp = G.input_name(g)
    x = graphs.synth_images(gold["images"], shapes[inp][1:], offset=gold["image_seed_offset"])
    net.set_quant_mode(OBSERVE)
    out = net.forward({inp: x})
    (sink, prob), = out.items()
    assert prob.dtype == np.float32 and prob.shape[0] == x.shape[0]
    ref = gold["ranges"]
    assert set(ref) <= set(net.ranges), set(ref) - set(net.ranges)
    for k, (lo, hi) in ref.items():
        glo, ghi = net.ranges[k]
        mag = max(abs(lo), abs(hi))
        assert abs(glo - lo) <= 1e-2 * mag and abs(ghi - hi) <= 1e-2 * mag, (k, (glo, ghi), (lo, hi))


@pytest.mark.gpu
def test_observe_then_quantize_alexnet():
    """qnet observe -> finalize -> quantized forward with the device-observed ranges
    (two calibration batches: observation only widens): the derived blob scales are
    within 2% of the ones the reference's ranges give, and the INT8 plan runs."""
    gold = _golden("alexnet")
    net, g, shapes = _net("alexnet")
    x = graphs.synth_images(gold["images"], shapes["data"][1:], offset=gold["image_seed_offset"])
    net.set_quant_mode(OBSERVE)
    net.forward({"data": x[:4]})
    net.forward({"data": x[4:]})
    net.finalize_quantizers()
    net.set_quant_mode(QUANTIZED)
    ours = net.forward({"data": x})["prob"]
    assert np.allclose(ours.sum(axis=1), 1.0, atol=1e-3)

    net2, _, _ = _net("alexnet")
    for k, (lo, hi) in gold["ranges"].items():
        net2.set_range(k, lo, hi)
    net2.finalize_quantizers()
    for b in net.blob_qv:
        a, r = net.blob_qv[b], net2.blob_qv[b]
        assert abs(a.scale - r.scale) <= 2e-2 * r.scale, (b, a.scale, r.scale)
