"""Parity at the benchmarked configuration (BASELINE configs[1] / configs[2]): the plan is
compiled at max_batch=256 and run on the full 256-image batch, exactly as bench.py times
it, and images {0-7, 248-255} are compared with the UNMODIFIED reference Net
(`Net::forward`, /root/reference/proj/src/net.cpp:305-330) on the same images.

At batch 256 every persistent GEMM CTA runs many tiles (AlexNet conv1 + relu1 + pool1 in
the front kernel: 3 456 pool rows in bands over 148 CTAs, ~48 conv rows each), so the
double-buffered TMEM accumulator phases, the input-row ring and the band hand-overs are
exercised; at batch 2 they are not.  Integer
checkpoints must be bit-identical; the FP32 softmax sink within 1 ulp."""
import json
import os

import numpy as np
import pytest

from oracle import ffi
from paper_2209_15427_b200 import graph as G
from paper_2209_15427_b200 import graphs
from paper_2209_15427_b200.net import QUANTIZED, Net

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
DT = {"fp32": 0, "fp16": 1, "int8": 2, "int16": 3}
PICK = list(range(8)) + list(range(248, 256))
THREADS = min(16, os.cpu_count() or 1)


def load_calib(model, precision):
    with open(os.path.join(HERE, "golden", f"{model}_{precision}_calib.json")) as f:
        return json.load(f)["ranges"]


def ref_nets(ref, g, precision, params, ranges, n=THREADS):
    from concurrent.futures import ThreadPoolExecutor

    def one(_):
        net = ref.net(json.dumps(g), precision)
        for k, v in params.items():
            net.set_param(k, v)
        for k, (lo, hi) in ranges.items():
            net.set_range(k, lo, hi)
        net.finalize()
        net.set_mode(3)
        return net

    with ThreadPoolExecutor(max_workers=n) as ex:
        return list(ex.map(one, range(n)))


def ref_forward(ref, g, precision, params, ranges, x, sink, per_bytes):
    nets = ref_nets(ref, g, precision, params, ranges)
    return ffi.forward_mt(nets, "data", x, sink, per_bytes)


def nhwc_rows(raw, lay, np_dtype, rows):
    n, h, w, cp, hh, hw, wx, es = lay
    a = raw.view(np_dtype).reshape(n, h + 2 * hh, w + 2 * hw + wx, cp)
    return a[rows, hh:hh + h, hw:hw + w, :]


@pytest.fixture(scope="module")
def alexnet256():
    if not ffi.have_reference():
        pytest.skip("needs oracle/_ref")
    import torch
    ref = ffi.Reference()
    g = graphs.alexnet(1)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    params = graphs.synth_params(g, shapes)
    ranges = load_calib("alexnet", "int8")
    ours = Net(G.override_precision(g, "int8"))
    for k, v in params.items():
        ours.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        ours.set_range(k, lo, hi)
    ours.finalize_quantizers()
    ours.set_quant_mode(QUANTIZED)
    B = 256
    x = graphs.synth_images(B, (3, 227, 227), offset=0)  # bench.py's rank-0 batch
    plan = ours.compile(B)
    xd = torch.from_numpy(x).cuda()
    od = torch.empty((B, 1000), dtype=torch.float32, device="cuda")
    plan.forward_device(xd.data_ptr(), od.data_ptr(), B)
    torch.cuda.synchronize()
    return ref, g, params, ranges, ours, plan, x, od.cpu().numpy()


@pytest.mark.parametrize("ck", ["pool1", "norm1", "relu2", "relu5", "pool5", "relu7", "fc8"])
def test_alexnet_int8_b256_checkpoints_bit_exact(alexnet256, ck):
    ref, g, params, ranges, ours, plan, x, _ = alexnet256
    names = [l["name"] for l in g["layers"]]
    prefix = {"name": "alexnet_prefix", "layers": g["layers"][: names.index(ck) + 1]}
    pr = {k: v for k, v in params.items() if k.split(".")[0] in names[: names.index(ck) + 1]}
    blob = ck if ck != "norm1" else "norm1__int8"
    raw, lay = plan.blob(blob)
    shp = G.infer_blobs(prefix)[prefix["layers"][-1]["top"][0]]["shape"]
    per = int(np.prod(shp[1:]))
    elem = 4 if ck == "norm1" else 1  # the reference prefix ends at the FP32 LRN
    theirs = ref_forward(ref, prefix, DT["int8"], pr, ranges, x[PICK], ck, per * elem)
    if ck == "norm1":
        theirs = ffi.Restatement().quantize(theirs.view(np.float32), ours.blob_qvals(blob), 2)
    theirs = theirs.reshape((len(PICK),) + tuple(shp[1:]))
    mine = nhwc_rows(raw, lay, np.uint8, PICK)
    if theirs.ndim == 4:
        theirs = np.transpose(theirs, (0, 2, 3, 1))
    else:
        theirs = theirs.reshape(len(PICK), 1, 1, -1)
    mine = mine[..., : theirs.shape[-1]]
    mism = int((mine != theirs).sum())
    assert mism == 0, f"{ck}: {mism} of {theirs.size} differ at batch 256"


def test_alexnet_int8_b256_prob_within_1ulp(alexnet256):
    ref, g, params, ranges, ours, plan, x, out = alexnet256
    theirs = ref_forward(ref, g, DT["int8"], params, ranges, x[PICK], "prob", 4000).view(np.float32)
    theirs = theirs.reshape(len(PICK), 1000)
    d = np.abs(out[PICK].view(np.int32).astype(np.int64) - theirs.view(np.int32).astype(np.int64))
    assert d.max() <= 1, d.max()


def test_alexnet_moe_int8_b256(reference):
    """AlexNet-MoE at batch 256: the MoE layer's quantized output (the sample-routed expert
    sub-batches, every expert's sub-batch many tiles deep) is bit-exact for 16 images, the
    sink within 1 ulp."""
    import torch
    from paper_2209_15427_b200.moe import MoeNet
    g = graphs.alexnet_moe(1)
    params = graphs.synth_params_moe(g)
    ranges = load_calib("alexnet_moe", "int8")
    ours = MoeNet(G.override_precision(g, "int8"))
    for k, v in params.items():
        ours.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        ours.set_range(k, lo, hi)
    ours.finalize_quantizers()
    ours.set_quant_mode(QUANTIZED)
    B = 256
    x = graphs.synth_images(B, (3, 227, 227), offset=0)
    xd = torch.from_numpy(x).cuda()
    od = torch.empty((B, 1000), dtype=torch.float32, device="cuda")
    ours.forward_device(xd.data_ptr(), od.data_ptr(), B)
    torch.cuda.synchronize()
    out = od.cpu().numpy()
    m_all = ours.moe_output(B)
    full = json.loads(reference.net(json.dumps(g), 2).graph_json())
    names = [l["name"] for l in full["layers"]]
    prefix = {"name": "moe_prefix", "layers": full["layers"][: names.index("moe") + 1],
              "range_aliases": full.get("range_aliases", {})}
    keep = {l["name"] for l in prefix["layers"]}
    pp = {k: v for k, v in params.items() if k.split(".")[0] in keep}
    per = m_all.shape[1]
    m_ref = ref_forward(reference, prefix, -1, pp, ranges, x[PICK], prefix["layers"][-1]["top"][0], per)
    m_ref = m_ref.reshape(len(PICK), per)
    assert np.array_equal(m_all[PICK], m_ref), int((m_all[PICK] != m_ref).sum())
    theirs = ref_forward(reference, g, 2, params, ranges, x[PICK], "prob", 4000).view(np.float32)
    d = np.abs(out[PICK].view(np.int32).astype(np.int64)
               - theirs.reshape(len(PICK), 1000).view(np.int32).astype(np.int64))
    assert d.max() <= 1, d.max()
