"""Whole-network parity on the B200: the compiled AlexNet INT8 plan against the
UNMODIFIED reference Net (oracle/_ref) on identical seeded weights, calibration and
images.  Integer blobs must be bit-identical at every checkpoint; the FP32 softmax
output may differ by 1 ulp (double exp in libm vs CUDA)."""
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


def load_calib(model, precision):
    with open(os.path.join(HERE, "golden", f"{model}_{precision}_calib.json")) as f:
        return json.load(f)["ranges"]


def nhwc_interior_to_nchw(raw, lay, np_dtype):
    n, h, w, cp, hh, hw, wx, es = lay
    a = raw.view(np_dtype).reshape(n, h + 2 * hh, w + 2 * hw + wx, cp)
    return a[:, hh:hh + h, hw:hw + w, :]


def ref_net(ref, g, precision, params, ranges):
    net = ref.net(json.dumps(g), DT[precision])
    for k, v in params.items():
        net.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        net.set_range(k, lo, hi)
    net.finalize()
    net.set_mode(3)
    return net


@pytest.fixture(scope="module")
def setup():
    if not ffi.have_reference():
        pytest.skip("needs oracle/_ref")
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
    return ref, g, params, ranges, ours


def test_finalize_matches_reference(setup):
    ref, g, params, ranges, ours = setup
    rn = ref_net(ref, g, "int8", params, ranges)
    for l in ours.graph["layers"]:
        if l["kind"] in ("conv", "inner_product"):
            w_ref, qv_ref = rn.param(l["name"] + ".weight")
            w_ours, dt, qv = ours.param(l["name"] + ".weight")
            assert qv.as_tuple() == qv_ref.as_tuple()
            assert np.array_equal(w_ours, w_ref), l["name"]
    for b in ours.blobs:
        q = ours.blob_qvals(b)
        if q is not None:
            assert q.as_tuple() == rn.blob_qvals(b).as_tuple(), b


@pytest.mark.parametrize("batch", [2, 7])
def test_alexnet_int8_bit_exact(setup, batch):
    """Checkpoints vs reference prefix nets.  pool1 is the front kernel's output (conv1 +
    relu1 + pool1 fused); batch 7 leaves the last image quad with one and a half pairs."""
    ref, g, params, ranges, ours = setup
    x = graphs.synth_images(batch, (3, 227, 227), offset=0)
    out = ours.forward({"data": x})["prob"]
    plan = ours.plan(batch)
    st = plan.stats()
    assert st["kernels_per_forward"] <= 16
    # checkpoints: reference prefix nets give the reference's blob at that point
    names = [l["name"] for l in g["layers"]]
    assert "conv_pool" in [s[1] for s in plan.steps()]
    for ck in ("pool1", "norm1", "relu2", "relu5", "pool5", "relu7", "fc8"):
        prefix = {"name": "alexnet_prefix", "layers": g["layers"][: names.index(ck) + 1]}
        pr = {k: v for k, v in params.items() if k.split(".")[0] in names[: names.index(ck) + 1]}
        rn = ref_net(ref, prefix, "int8", pr, ranges)
        res = rn.forward("data", x)
        (arr, dt, qv), = [v for k, v in res.items()]
        blob = ck if ck != "norm1" else "norm1__int8"
        if dt == 0:  # the prefix ends at the FP32 LRN: apply the full net's norm1_to_int8
            arr = ffi.Restatement().quantize(arr, ours.blob_qvals(blob), 2)
        got = plan.blob(blob)
        assert got is not None, blob
        raw, lay = got
        mine = nhwc_interior_to_nchw(raw, lay, np.uint8)
        theirs = arr.reshape(batch, lay[3] if arr.ndim == 2 else arr.shape[1], *(arr.shape[2:] or (1, 1)))
        if arr.ndim == 4:
            theirs = np.transpose(arr, (0, 2, 3, 1))
        else:
            theirs = arr.reshape(batch, 1, 1, -1)
        mine = mine[..., : theirs.shape[-1]]
        mism = int((mine != theirs).sum())
        assert mism == 0, f"{ck}: {mism} of {theirs.size} differ"
    rn = ref_net(ref, g, "int8", params, ranges)
    res = rn.forward("data", x)
    prob_ref = res["prob"][0]
    d = np.abs(out.view(np.int32).astype(np.int64) - prob_ref.view(np.int32).astype(np.int64))
    assert d.max() <= 1, d.max()


def test_host_buffer_pipeline_matches_device_forward(setup):
    """qnb_plan_forward with host buffers cuts the batch into chunks whose H2D copies
    overlap the previous chunk's forward; pinned (CUDA-graph) and pageable (eager)
    sources must give exactly the device-resident result."""
    import torch
    ref, g, params, ranges, ours = setup
    batch = 100  # 3 chunks of 34 / 34 / 32
    x = graphs.synth_images(batch, (3, 227, 227), offset=500)
    plan = ours.compile(batch)
    xd = torch.from_numpy(x).cuda()
    od = torch.empty((batch, 1000), dtype=torch.float32, device="cuda")
    plan.forward_device(xd.data_ptr(), od.data_ptr(), batch)
    torch.cuda.synchronize()
    want = od.cpu().numpy()
    xp = torch.from_numpy(x).pin_memory()
    op = torch.empty((batch, 1000), dtype=torch.float32).pin_memory()
    for _ in range(2):  # capture, then replay
        op.zero_()
        plan.forward_device(xp.data_ptr(), op.data_ptr(), batch, in_host=True, out_host=True)
        torch.cuda.synchronize()
        assert np.array_equal(op.numpy(), want)
    got = plan.forward_host(x)  # pageable numpy buffers
    assert np.array_equal(got, want)


def test_inspect_blobs_stay_addressable(setup):
    """Graph::inspect (include/qnet/graph.hpp:96): inspected blobs are never fused away.
    conv1 (normally fused with relu1), pool1 (normally inside the pool+LRN kernel) and
    fc8__fp32 (normally inside the softmax) get their own buffers; their contents equal
    the reference's blob and the network output is unchanged."""
    ref, g, params, ranges, ours = setup
    batch = 2
    x = graphs.synth_images(batch, (3, 227, 227), offset=3)
    gi = G.override_precision(g, "int8")
    gi["inspect"] = ["conv1", "pool1", "fc8__fp32"]
    net = Net(gi)
    for k, (arr, dt, qv) in ours.params.items():
        net.set_param(k, arr, dt, qv)
    net.blob_qv = dict(ours.blob_qv)
    net.set_quant_mode(QUANTIZED)
    out = net.forward({"data": x})["prob"]
    assert np.array_equal(out, ours.forward({"data": x})["prob"])
    plan = net.plan(batch)
    assert plan.stats()["kernels_per_forward"] > ours.plan(batch).stats()["kernels_per_forward"]
    names = [l["name"] for l in g["layers"]]
    for ck in ("conv1", "pool1"):
        prefix = {"name": "alexnet_prefix", "layers": g["layers"][: names.index(ck) + 1]}
        pr = {k: v for k, v in params.items() if k.split(".")[0] in names[: names.index(ck) + 1]}
        (arr, dt, qv), = ref_net(ref, prefix, "int8", pr, ranges).forward("data", x).values()
        raw, lay = plan.blob(ck)
        mine = nhwc_interior_to_nchw(raw, lay, np.uint8)[..., : arr.shape[1]]
        assert np.array_equal(mine, np.transpose(arr, (0, 2, 3, 1))), ck
    raw, lay = plan.blob("fc8__fp32")
    fc8 = nhwc_interior_to_nchw(raw, lay, np.float32).reshape(batch, -1)[:, :1000]
    e = np.exp(fc8.astype(np.float64) - fc8.max(axis=1, keepdims=True))
    assert np.allclose(e / e.sum(axis=1, keepdims=True), out, rtol=1e-5, atol=1e-9)


def test_device_resident_batch(setup):
    """qnb_plan_forward_dyn: a plan launched at its capacity with the batch in device
    memory (the MoE experts' routed sub-batches) gives exactly the host-batch forward for
    the live images and leaves the rows past the device batch untouched."""
    import torch
    ref, g, params, ranges, ours = setup
    cap = 64
    plan = ours.compile(cap, use_cuda_graph=False)
    x = graphs.synth_images(cap, (3, 227, 227), offset=700)
    xd = torch.from_numpy(x).cuda()
    for n in (37, 1, 64, 2):
        want = torch.empty((n, 1000), dtype=torch.float32, device="cuda")
        plan.forward_device(xd.data_ptr(), want.data_ptr(), n)
        got = torch.full((cap, 1000), -7.0, dtype=torch.float32, device="cuda")
        dyn = torch.tensor([n], dtype=torch.int32, device="cuda")
        plan.forward_dyn(xd.data_ptr(), got.data_ptr(), cap, dyn.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(got[:n], want), n
        assert bool((got[n:] == -7.0).all()), n


def test_front_zero_point_row_fallback(setup, monkeypatch):
    """The conv1 front kernel runs its A operand as s8 (w - zW) when every weight fits;
    otherwise an extra A row of zW gives zW * rowsum, which the lane quarter holding it
    hands to the others through shared memory.  Both forms give the same pool1 bytes and
    the same network output (the reference comparison is test_alexnet_int8_bit_exact)."""
    ref, g, params, ranges, ours = setup
    batch = 9
    x = graphs.synth_images(batch, (3, 227, 227), offset=41)
    pa = ours.plan(batch)
    out_sa = ours.forward({"data": x})["prob"]
    pool_sa = pa.blob("pool1")[0].copy()
    monkeypatch.setenv("QNB_FRONT_NO_SA", "1")
    net = Net(G.override_precision(g, "int8"))
    for k, (arr, dt, qv) in ours.params.items():
        net.set_param(k, arr, dt, qv)
    net.blob_qv = dict(ours.blob_qv)
    net.set_quant_mode(QUANTIZED)
    out_row = net.forward({"data": x})["prob"]
    pb = net.plan(batch)
    assert "conv_pool" in [s[1] for s in pb.steps()]
    assert np.array_equal(pb.blob("pool1")[0], pool_sa)
    assert np.array_equal(out_row, out_sa)
