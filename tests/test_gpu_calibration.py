"""OBSERVE-mode calibration on the device (Net::forward with QuantMode::OBSERVE,
src/net.cpp:305-330, observe() src/quantizer.cpp:58-68) against the ranges the
UNMODIFIED reference recorded over the same seeded images (tests/golden/*_calib.json,
made by tests/golden/make_calibration.py), and PSEUDO-mode forwards against the
reference's.  Calibration plans run the FP32 conv / inner products in the reference's
exact arithmetic (QNB_PLAN_EXACT_FLOAT), so both are bit-identical."""
import json
import os

import numpy as np
import pytest

from paper_2209_15427_b200 import graph as G
from paper_2209_15427_b200 import graphs
from paper_2209_15427_b200.net import OBSERVE, PSEUDO, QUANTIZED, Net

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
        assert tuple(net.ranges[k]) == (lo, hi), (k, net.ranges[k], (lo, hi))


@pytest.mark.gpu
def test_observe_then_quantize_alexnet():
    """qnet observe -> finalize -> quantized forward with the device-observed ranges
    (two calibration batches: observation only widens): the derived blob grids are
    exactly the ones the reference's ranges give, and the INT8 plan runs."""
    gold = _golden("alexnet")
    net, g, shapes = _net("alexnet")
    x = graphs.synth_images(gold["images"], shapes["data"][1:], offset=gold["image_seed_offset"])
    net.set_quant_mode(OBSERVE)
    net.forward({"data": x[:3]})
    net.forward({"data": x[3:]})
    net.finalize_quantizers()
    net.set_quant_mode(QUANTIZED)
    ours = net.forward({"data": x})["prob"]
    assert np.allclose(ours.sum(axis=1), 1.0, atol=1e-3)

    net2, _, _ = _net("alexnet")
    for k, (lo, hi) in gold["ranges"].items():
        net2.set_range(k, lo, hi)
    net2.finalize_quantizers()
    for b in net.blob_qv:
        assert net.blob_qv[b].as_tuple() == net2.blob_qv[b].as_tuple(), b


def _finalized(model):
    net, g, shapes = _net(model)
    for k, (lo, hi) in _golden(model)["ranges"].items():
        net.set_range(k, lo, hi)
    net.finalize_quantizers()
    return net, g, shapes


def test_pseudo_graph_fake_quantizes_every_declared_top():
    from paper_2209_15427_b200 import ops
    net, _, _ = _net("alexnet")
    for k, (lo, hi) in _golden("alexnet")["ranges"].items():
        net.set_range(k, lo, hi)
    for b, info in net.blobs.items():  # the blob half of finalize_quantizers (host only)
        if info["dtype"] in G.QUANT:
            r = net.range(b)
            net.blob_qv[b] = ops.estimate_from_observation(r[0], r[1], G.DTYPE_CODE[info["dtype"]])
    pg, sink = net.pseudo_graph()
    assert sink == "prob"
    fq = [l for l in pg["layers"] if l["kind"] == "quantizer"]
    assert all(l["bottom_data_type"] == l["top_data_type"] == G.FP32 for l in fq)
    # one fake-quant per non-FP32 top of the typed graph (QUANTIZER tops included)
    want = [l["top"][0] for l in net.graph["layers"] if l["top_data_type"] != G.FP32]
    assert [l["top"][0] for l in fq] == [b + "__pseudo" for b in want]
    assert fq[0]["bottom"] == ["data"] and fq[0]["pseudo_qv"] is net.blob_qv["data__int8"]
    conv2 = next(l for l in pg["layers"] if l.get("name") == "conv2")
    assert conv2["bottom"] == ["norm1__int8__pseudo"]


def _ref_pseudo(model, x, prefix_to=None):
    from oracle import ffi
    if not ffi.have_reference():
        pytest.skip("needs oracle/_ref")
    g = graphs.MODELS[model](1)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    params = graphs.synth_params(g, shapes)
    if prefix_to is not None:
        names = [l["name"] for l in g["layers"]]
        keep = names[: names.index(prefix_to) + 1]
        g = {"name": "prefix", "layers": g["layers"][: len(keep)]}
        params = {k: v for k, v in params.items() if k.split(".")[0] in keep}
    rn = ffi.Reference().net(json.dumps(g), 2)
    for k, v in params.items():
        rn.set_param(k, v)
    for k, (lo, hi) in _golden(model)["ranges"].items():
        rn.set_range(k, lo, hi)
    rn.finalize()
    rn.set_mode(2)  # PSEUDO
    (arr, dt, _), = rn.forward(G.input_name(g), x).values()
    return arr


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["lenet5", "vgg16_32", "alexnet"])
def test_pseudo_matches_reference(model):
    """PSEUDO forward (exact FP32 contractions + fake-quant kernels) against the
    reference's PSEUDO forward: bit-identical."""
    net, g, shapes = _finalized(model)
    inp = G.input_name(g)
    x = graphs.synth_images(2, shapes[inp][1:], offset=41)
    net.set_quant_mode(PSEUDO)
    out = net.forward({inp: x})
    (sink, prob), = out.items()
    theirs = _ref_pseudo(model, x)
    assert prob.dtype == np.float32
    assert np.array_equal(prob.reshape(theirs.shape), theirs)
