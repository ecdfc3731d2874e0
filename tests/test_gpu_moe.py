"""AlexNet-MoE INT8 (BASELINE configs[2]) on the B200 vs the
unmodified reference qnet::Net: the MoE layer's quantized output is bit-exact and the
softmax sink is within 1 ulp (libm exp vs device exp in the FP32 island)."""
import json
import os

import numpy as np
import pytest

from paper_2209_15427_b200 import graph as G
from paper_2209_15427_b200 import graphs
from paper_2209_15427_b200.net import QUANTIZED

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def setup(reference):
    g = graphs.alexnet_moe(1)
    params = graphs.synth_params_moe(g)
    with open(os.path.join(ROOT, "tests", "golden", "alexnet_moe_int8_calib.json")) as f:
        ranges = json.load(f)["ranges"]
    return g, params, ranges


def ref_net(reference, graph_json, params, ranges, precision):
    net = reference.net(graph_json, precision)
    for k, v in params.items():
        net.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        net.set_range(k, lo, hi)
    net.finalize()
    net.set_mode(3)
    return net


def our_net(g, params, ranges):
    from paper_2209_15427_b200.moe import MoeNet
    net = MoeNet(G.override_precision(g, "int8"))
    for k, v in params.items():
        net.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        net.set_range(k, lo, hi)
    net.finalize_quantizers()
    net.set_quant_mode(QUANTIZED)
    return net


def test_alexnet_moe_int8_matches_reference(reference, setup):
    import torch
    g, params, ranges = setup
    batch = 3
    x = graphs.synth_images(batch, (3, 227, 227), offset=0)
    ours = our_net(g, params, ranges)
    out = ours.forward({"data": x})["prob"]
    counts = ours.last_stats["counts"]
    assert counts.sum() == batch * 4

    rn = ref_net(reference, json.dumps(g), params, ranges, 2)
    full = json.loads(rn.graph_json())
    prob_ref = rn.forward("data", x)["prob"][0]
    d = np.abs(out.view(np.int32).astype(np.int64) - prob_ref.view(np.int32).astype(np.int64))
    assert d.max() <= 1, d.max()

    # the MoE layer's own quantized output, bit for bit (reference prefix net ending at it)
    names = [l["name"] for l in full["layers"]]
    prefix = {"name": "moe_prefix", "layers": full["layers"][: names.index("moe") + 1],
              "range_aliases": full.get("range_aliases", {})}
    keep = {l["name"] for l in prefix["layers"]}
    pp = {k: v for k, v in params.items() if k.split(".")[0] in keep}
    rp = ref_net(reference, json.dumps(prefix), pp, ranges, -1)
    (m_ref, dt, qv), = rp.forward("data", x).values()
    assert dt == 2
    m_ours = ours.moe_output(batch).reshape(m_ref.shape)
    assert np.array_equal(m_ours, m_ref), int((m_ours != m_ref).sum())
    torch.cuda.synchronize()


def test_alexnet_moe_host_buffers_match_device_path(setup):
    """forward_device with pinned host input / output (the trunk plan pipelines the H2D
    copy chunk by chunk, the tail plan copies the result back) gives the device-buffer
    result bit for bit, at a batch large enough to be split into several chunks."""
    import torch
    g, params, ranges = setup
    batch = 96
    x = graphs.synth_images(batch, (3, 227, 227), offset=300)
    ours = our_net(g, params, ranges)
    xd = torch.from_numpy(x).cuda()
    od = torch.empty((batch, 1000), dtype=torch.float32, device="cuda")
    ours.forward_device(xd.data_ptr(), od.data_ptr(), batch)
    torch.cuda.synchronize()
    want = od.cpu().numpy()
    xp = torch.from_numpy(x).pin_memory()
    op = torch.empty((batch, 1000), dtype=torch.float32).pin_memory()
    for _ in range(2):
        op.zero_()
        ours.forward_device(xp.data_ptr(), op.data_ptr(), batch, in_host=True, out_host=True)
        torch.cuda.synchronize()
        assert np.array_equal(op.numpy(), want)


def test_alexnet_moe_noisy_gating_matches_reference(reference, setup):
    """Gating noise on (MoeLayerParams::noise_enabled, src/moe.cpp:53-71, 92-95) with
    non-zero W_b / W_c, through the device-driven MoE plan: the noise table is drawn with
    the reference's own arithmetic, so routing and the MoE output are bit-identical."""
    g, params, ranges = setup
    g = json.loads(json.dumps(g))
    moe = next(l for l in g["layers"] if l["kind"] == "moe")
    moe["moe"]["noise_enabled"] = True
    moe["moe"]["seed"] = 12345
    params = dict(params)
    rng = np.random.default_rng(77)
    N, D = params["moe.gate_a"].shape
    params["moe.gate_b"] = rng.uniform(-0.3, 0.3, (N, D)).astype(np.float32)
    params["moe.gate_c"] = rng.uniform(-0.5, 0.5, (N,)).astype(np.float32)
    batch = 3
    x = graphs.synth_images(batch, (3, 227, 227), offset=40)
    ours = our_net(g, params, ranges)
    out = ours.forward({"data": x})["prob"]
    rn = ref_net(reference, json.dumps(g), params, ranges, 2)
    full = json.loads(rn.graph_json())
    prob_ref = rn.forward("data", x)["prob"][0]
    d = np.abs(out.view(np.int32).astype(np.int64) - prob_ref.view(np.int32).astype(np.int64))
    assert d.max() <= 1, d.max()
    names = [l["name"] for l in full["layers"]]
    prefix = {"name": "moe_prefix", "layers": full["layers"][: names.index("moe") + 1],
              "range_aliases": full.get("range_aliases", {})}
    keep = {l["name"] for l in prefix["layers"]}
    pp = {k: v for k, v in params.items() if k.split(".")[0] in keep}
    (m_ref, dt, qv), = ref_net(reference, json.dumps(prefix), pp, ranges, -1).forward("data", x).values()
    assert np.array_equal(ours.moe_output(batch).reshape(m_ref.shape), m_ref)


def test_moe_plan_counts_and_graph_replay(setup):
    """The MoE plan replays one CUDA graph; routing counts come back only on request
    (qnb_moe_plan_status) and always sum to batch * top_k; a replay at another batch
    size (new graph) and back gives identical outputs."""
    import torch
    g, params, ranges = setup
    ours = our_net(g, params, ranges)
    outs = {}
    for batch in (40, 17, 40):
        x = graphs.synth_images(batch, (3, 227, 227), offset=900)
        xd = torch.from_numpy(x).cuda()
        od = torch.empty((batch, 1000), dtype=torch.float32, device="cuda")
        ours.forward_device(xd.data_ptr(), od.data_ptr(), batch)
        counts = ours.last_stats["counts"]
        assert counts.sum() == batch * 4 and (counts >= 0).all()
        o = od.cpu().numpy()
        if batch in outs:
            assert np.array_equal(outs[batch], o)
        outs[batch] = o
    assert np.array_equal(outs[17], outs[40][:17])  # per-sample independence (same seeds)


def test_group_world1_forward_and_collectives(setup):
    """qnb_group_* with one rank (NCCL communicator of size 1 on this GPU): the grouped
    forward equals the plan's own forward, all-gather and all-to-all move the bytes."""
    import torch
    from paper_2209_15427_b200.group import Group
    from paper_2209_15427_b200.net import QUANTIZED, Net
    g = graphs.alexnet(1)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    params = graphs.synth_params(g, shapes)
    with open(os.path.join(ROOT, "tests", "golden", "alexnet_int8_calib.json")) as f:
        ranges = json.load(f)["ranges"]
    net = Net(G.override_precision(g, "int8"))
    for k, v in params.items():
        net.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        net.set_range(k, lo, hi)
    net.finalize_quantizers()
    net.set_quant_mode(QUANTIZED)
    B = 8
    plan = net.compile(B)
    x = torch.from_numpy(graphs.synth_images(B, (3, 227, 227), offset=11)).cuda()
    want = torch.empty((B, 1000), dtype=torch.float32, device="cuda")
    plan.forward_device(x.data_ptr(), want.data_ptr(), B)
    grp = Group(1, 0, Group.unique_id(), torch.cuda.current_device())
    got = torch.zeros((B, 1000), dtype=torch.float32, device="cuda")
    grp.forward(plan, x.data_ptr(), B, got.data_ptr(), 4000, torch.cuda.current_stream().cuda_stream)
    src = torch.arange(64, dtype=torch.uint8, device="cuda")
    dst = torch.zeros(64, dtype=torch.uint8, device="cuda")
    grp.alltoallv(src.data_ptr(), [0], [64], dst.data_ptr(), [0], [64], torch.cuda.current_stream().cuda_stream)
    ag = torch.zeros(64, dtype=torch.uint8, device="cuda")
    grp.allgather(src.data_ptr(), ag.data_ptr(), 64, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert torch.equal(dst, src) and torch.equal(ag, src)
