"""QCNM model store (src/model_store.cpp, Net::to_model / load_weights src/net.cpp:546-619)
through the qnb_model_* C-ABI: files written by the UNMODIFIED reference load here and
save back byte-identical; the reference's error messages; and (GPU) a plan compiled from
a loaded file runs bit-exact against the reference Net loaded from the same file."""
import json
import os

import numpy as np
import pytest

from oracle import ffi
from paper_2209_15427_b200 import graph as G
from paper_2209_15427_b200 import graphs
from paper_2209_15427_b200._lib import QnbError
from paper_2209_15427_b200.model_store import Model, ParamRecord, load_model, save_model
from paper_2209_15427_b200.net import QUANTIZED, Net

HERE = os.path.dirname(os.path.abspath(__file__))
DT = {"fp32": 0, "int8": 2, "int16": 3}


def _ref():
    if not ffi.have_reference():
        pytest.skip("needs oracle/_ref")
    return ffi.Reference()


def _ranges(model):
    with open(os.path.join(HERE, "golden", f"{model}_int8_calib.json")) as f:
        return json.load(f)["ranges"]


def _ref_file(ref, model, precision, path, finalize=True):
    g = graphs.MODELS[model](1)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    rn = ref.net(json.dumps(g), DT[precision] if precision != "fp32" else -1)
    for k, v in graphs.synth_params(g, shapes).items():
        rn.set_param(k, v)
    for k, (lo, hi) in _ranges(model).items():
        rn.set_range(k, lo, hi)
    if finalize:
        rn.finalize()
    rn.save(str(path))
    return g, rn


@pytest.mark.parametrize("model,precision,finalize", [("lenet5", "int8", True), ("alexnet", "int8", True),
                                                      ("alexnet", "fp32", False), ("vgg16_32", "int16", True)])
def test_reference_file_round_trips_byte_identical(tmp_path, model, precision, finalize):
    ref = _ref()
    p1, p2 = tmp_path / "ref.qcnm", tmp_path / "ours.qcnm"
    g, _ = _ref_file(ref, model, precision, p1, finalize)
    rn = ref.net(json.dumps(g), DT[precision] if precision != "fp32" else -1)
    rn.load(str(p1))  # the reference's own view of the file (float-narrowed qvals)
    net = Net(G.override_precision(g, precision) if precision != "fp32" else g)
    m = load_model(str(p1))
    net.load_weights(m)
    # parameters and quantizer values are the reference's
    for r in m.records:
        if r.name.startswith("blob:"):
            continue
        arr, qv = rn.param(r.name)
        mine, dt, mqv = net.param(r.name)
        assert np.array_equal(mine, arr), r.name
        assert (mqv is None) == (qv is None)
        if qv is not None:
            assert mqv.as_tuple() == qv.as_tuple(), r.name
    save_model(net.to_model(), str(p2))
    assert p1.read_bytes() == p2.read_bytes()


def test_payloads_are_views_into_the_mapping(tmp_path):
    p = tmp_path / "m.qcnm"
    w = np.arange(24, dtype=np.float32).reshape(2, 3, 4)
    save_model(Model([ParamRecord("fc.weight", 0, w.shape, payload=w.view(np.uint8).reshape(-1)),
                      ParamRecord("blob:data", 0, (0,), -1.5, 2.5)]), str(p))
    m = load_model(str(p))
    a = m.records[0].array()
    assert not a.flags.owndata and not a.flags.writeable
    assert np.array_equal(a, w)
    assert m.records[1].extents == (0,) and m.records[1].payload.size == 0
    assert (m.records[1].f_min, m.records[1].f_max) == (-1.5, 2.5)


def test_payload_views_outlive_the_model(tmp_path):
    """The mapping is released only when the last view into it is gone: records taken
    from a temporary Model stay readable (the views hold the mapping alive)."""
    import gc
    p = tmp_path / "m.qcnm"
    w = np.arange(4096, dtype=np.float32)
    save_model(Model([ParamRecord("fc.weight", 0, w.shape, payload=w.view(np.uint8).reshape(-1))]), str(p))
    recs = load_model(str(p)).records
    gc.collect()
    assert float(recs[0].array().sum()) == float(w.sum())
    arr = load_model(str(p)).records[0].array()
    gc.collect()
    assert np.array_equal(arr, w)


def test_huge_record_count_is_a_truncated_file(tmp_path):
    """An untrusted u32 record count must not turn into a huge reservation (the
    reference's reader reports the file as truncated)."""
    bad = tmp_path / "count.qcnm"
    bad.write_bytes(b"QCNM\x01\xff\xff\xff\xff")
    with pytest.raises(QnbError, match="truncated model file") as e:
        load_model(str(bad))
    assert e.value.status == 11


def test_load_errors_carry_reference_messages(tmp_path):
    with pytest.raises(QnbError, match="cannot read: "):
        load_model(str(tmp_path / "missing.qcnm"))
    bad = tmp_path / "bad.qcnm"
    bad.write_bytes(b"NOPE\x01\x00\x00\x00\x00")
    with pytest.raises(QnbError, match="not a model file") as e:
        load_model(str(bad))
    assert e.value.status == 11
    good = tmp_path / "good.qcnm"
    w = np.ones(16, np.float32)
    save_model(Model([ParamRecord("a.weight", 0, (16,), payload=w.view(np.uint8))]), str(good))
    trunc = tmp_path / "trunc.qcnm"
    trunc.write_bytes(good.read_bytes()[:-5])
    with pytest.raises(QnbError, match="truncated model file"):
        load_model(str(trunc))
    tag = bytearray(good.read_bytes())
    tag[5 + 4 + 2 + len("a.weight")] = 9  # dtype tag past INT16Q
    (tmp_path / "tag.qcnm").write_bytes(bytes(tag))
    with pytest.raises(QnbError, match="not a model file"):
        load_model(str(tmp_path / "tag.qcnm"))
    with pytest.raises(QnbError, match="payload size mismatch: x"):
        save_model(Model([ParamRecord("x", 0, (4,), payload=np.zeros(3, np.uint8))]), str(tmp_path / "y"))


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["lenet5", "alexnet"])
def test_plan_from_loaded_file_bit_exact(tmp_path, model):
    """`qnet infer` flow (tools/qnet_main.cpp:163-175): load the model, finalize,
    QUANTIZED forward — ours from the mapped file vs the reference Net from the same file."""
    ref = _ref()
    p = tmp_path / "m.qcnm"
    g, _ = _ref_file(ref, model, "int8", p)
    net = Net(G.override_precision(g, "int8"))
    net.load_weights(load_model(str(p)))
    net.finalize_quantizers()
    net.set_quant_mode(QUANTIZED)
    inp = G.input_name(g)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    x = graphs.synth_images(2, shapes[inp][1:], offset=77)
    (name, mine), = net.forward({inp: x}).items()
    rn = ref.net(json.dumps(g), 2)
    rn.load(str(p))
    rn.finalize()
    rn.set_mode(3)
    arr, dt, _ = rn.forward(inp, x)[name]
    if dt == 0:
        d = np.abs(mine.view(np.int32).astype(np.int64) - arr.view(np.int32).astype(np.int64))
        assert d.max() <= 1
    else:
        assert np.array_equal(mine, arr)
