"""Op-level parity on the B200: every sm_100a kernel against the CPU oracle.

The checker is the compiled reference (oracle/_ref) when present, else the pinned
plain-C restatement.  Integer outputs must be bit-exact; float islands that go
through libm (LRN pow, softmax exp) are allowed 1 ulp on a tiny fraction of
elements; tensor-core float convolutions use the north-star tolerance
(max-abs <= 1e-2 x output range).
"""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import pytest

from paper_2209_15427_b200 import ops
from paper_2209_15427_b200._lib import FP16, FP32, INT8Q, INT16Q

pytestmark = pytest.mark.gpu


def qv_of(oracle_impl, lo, hi, dt=INT8Q):
    return oracle_impl.estimate_params(lo, hi, dt)


def assert_bits_equal(a, b, what=""):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
        bad = np.argwhere(a != b)
        msg = f"{what}: {len(bad)} of {a.size} differ; first {bad[:8].tolist()} ours {a[tuple(bad[:8].T)]} " \
              f"oracle {b[tuple(bad[:8].T)]}"
        raise AssertionError(msg)


def ulp_diff(a, b):
    ai = a.view(np.int32).astype(np.int64)
    bi = b.view(np.int32).astype(np.int64)
    return np.abs(ai - bi)


# ------------------------------------------------------------ elementwise
@pytest.mark.parametrize("dtype", [INT8Q, INT16Q])
def test_quantize_dequantize(oracle_impl, dtype):
    rng = np.random.default_rng(10)
    qv = qv_of(oracle_impl, -3.3, 7.1, dtype)
    x = rng.uniform(-10, 12, 1 << 20).astype(np.float32)
    # exact ties of x / scale and specials
    k = np.arange(-50, 50, dtype=np.float64)
    ties = ((k + 0.5) * qv.scale).astype(np.float32)
    x[: ties.size] = ties
    x[-5:] = [np.nan, np.inf, -np.inf, 0.0, -0.0]
    ours = ops.quantize(x, qv, dtype)
    assert_bits_equal(ours, oracle_impl.quantize(x, qv, dtype), "quantize")
    back = ops.dequantize(ours, dtype, qv)
    assert_bits_equal(back, oracle_impl.dequantize(ours, dtype, qv), "dequantize")


def test_requantize_and_relu_quant(oracle_impl):
    rng = np.random.default_rng(11)
    for trial in range(12):
        din = INT8Q if trial % 3 else INT16Q
        dout = INT8Q if trial % 2 else INT16Q
        qi = qv_of(oracle_impl, -rng.uniform(0.1, 5), rng.uniform(0.1, 5), din)
        qo = qv_of(oracle_impl, -rng.uniform(0.0, 5), rng.uniform(0.1, 9), dout)
        sb = 31 if dout == INT8Q else 15
        rq = oracle_impl.scale_quant_vals(qi, qo, sb)
        q = rng.integers(0, 256 if din == INT8Q else 65536, 100_000).astype(np.uint8 if din == INT8Q else np.uint16)
        from paper_2209_15427_b200._lib import Requant
        ours = ops.requantize(q, din, Requant(*rq.as_tuple()), dout)
        from oracle.ffi import Restatement
        assert_bits_equal(ours, Restatement().requantize(q, din, rq, dout), "requantize")
        if din == dout:
            r = ops.relu_quant(q, din, Requant(*rq.as_tuple()))
            assert_bits_equal(r, oracle_impl.relu_quant(q, din, rq), "relu_quant")


def test_relu_float_and_cast(oracle_impl):
    rng = np.random.default_rng(12)
    x = rng.normal(0, 100, 300_000).astype(np.float32)
    x[:3] = [np.nan, -0.0, np.inf]
    for slope in (0.0, 0.1):
        assert_bits_equal(ops.relu_float(x, FP32, slope), oracle_impl.relu_float(x, FP32, slope), "relu32")
    h = oracle_impl.cast_float(x, FP32, FP16)
    assert_bits_equal(ops.cast_float(x, FP32, FP16), h, "cast f32->f16")
    assert_bits_equal(ops.cast_float(h, FP16, FP32), oracle_impl.cast_float(h, FP16, FP32), "cast f16->f32")
    assert_bits_equal(ops.relu_float(h, FP16, 0.0), oracle_impl.relu_float(h, FP16, 0.0), "relu16")


@pytest.mark.parametrize("dtype", [INT8Q, INT16Q, FP32, FP16])
@pytest.mark.parametrize("shape,k,s", [((2, 96, 55, 55), 3, 2), ((3, 5, 13, 13), 3, 2), ((2, 7, 8, 9), 2, 2)])
def test_pool_max(oracle_impl, dtype, shape, k, s):
    rng = np.random.default_rng(13)
    if dtype in (INT8Q, INT16Q):
        x = rng.integers(0, 256 if dtype == INT8Q else 65536, shape).astype(np.uint8 if dtype == INT8Q else np.uint16)
    else:
        x = rng.normal(0, 1, shape).astype(np.float32)
        if dtype == FP16:
            x = oracle_impl.cast_float(x, FP32, FP16)
    assert_bits_equal(ops.pool_max(x, dtype, k, s), oracle_impl.pool_max(x, dtype, k, s), "pool")


def test_lrn_alexnet_shapes(oracle_impl):
    rng = np.random.default_rng(14)
    for shape in ((2, 96, 27, 27), (2, 256, 13, 13)):
        x = np.abs(rng.normal(0, 40, shape)).astype(np.float32)
        a, b = ops.lrn(x), oracle_impl.lrn(x)
        d = ulp_diff(a, b)
        assert d.max() <= 1, d.max()
        assert (d > 0).mean() < 1e-4, (d > 0).mean()


def test_softmax(oracle_impl):
    rng = np.random.default_rng(15)
    x = rng.normal(0, 4, (256, 1000)).astype(np.float32)
    d = ulp_diff(ops.softmax(x), oracle_impl.softmax(x))
    assert d.max() <= 1 and (d > 0).mean() < 1e-3


# ------------------------------------------------------- contractions (tcgen05)
def _conv_case(oracle_impl, rng, N, C, H, W, cp, dtype):
    G = cp.get("groups", 1)
    xf = rng.uniform(-2, 2, (N, C, H, W)).astype(np.float32)
    wf = rng.uniform(-0.5, 0.5, (cp["out_channels"], C // G, cp["kernel_h"], cp["kernel_w"])).astype(np.float32)
    bias = rng.uniform(-0.3, 0.3, cp["out_channels"]).astype(np.float32)
    if dtype == INT8Q:
        qx, qw = qv_of(oracle_impl, -2, 2.5), qv_of(oracle_impl, -0.5, 0.55)
        K = C // G * cp["kernel_h"] * cp["kernel_w"]
        span = 0.4 * np.sqrt(K)
        qo = qv_of(oracle_impl, -span, span * 1.1)
        x, w = oracle_impl.quantize(xf, qx, INT8Q), oracle_impl.quantize(wf, qw, INT8Q)
        ours = ops.conv_forward(x, INT8Q, w, INT8Q, bias, cp, qx, qw, qo)
        theirs = oracle_impl.conv_forward(x, INT8Q, w, INT8Q, bias, cp, qx, qw, qo)
        assert_bits_equal(ours, theirs, f"conv int8 {cp}")
        assert len(np.unique(theirs)) > 16  # the grid is exercised, not saturated
    else:
        x = xf if dtype == FP32 else oracle_impl.cast_float(xf, FP32, FP16)
        ours = ops.conv_forward(x, dtype, wf, FP32, bias, cp)
        theirs = oracle_impl.conv_forward(x, dtype, wf, FP32, bias, cp)
        if dtype == FP16:
            ours = oracle_impl.cast_float(ours, FP16, FP32)
            theirs = oracle_impl.cast_float(theirs, FP16, FP32)
        rng_ = float(theirs.max() - theirs.min())
        err = float(np.abs(ours - theirs).max())
        assert err <= 1e-2 * rng_, (err, rng_)


CONV_CASES = [
    # (N, C, H, W, conv params) — AlexNet conv1..conv5 geometry at small batch, then edge cases
    (1, 3, 227, 227, dict(out_channels=96, kernel_h=11, kernel_w=11, stride_h=4, stride_w=4)),
    (1, 96, 27, 27, dict(out_channels=256, kernel_h=5, kernel_w=5, pad_h=2, pad_w=2, groups=2)),
    (1, 256, 13, 13, dict(out_channels=384, kernel_h=3, kernel_w=3, pad_h=1, pad_w=1)),
    (1, 384, 13, 13, dict(out_channels=384, kernel_h=3, kernel_w=3, pad_h=1, pad_w=1, groups=2)),
    (2, 384, 13, 13, dict(out_channels=256, kernel_h=3, kernel_w=3, pad_h=1, pad_w=1, groups=2)),
    (3, 16, 9, 11, dict(out_channels=20, kernel_h=3, kernel_w=3, stride_h=2, stride_w=1, pad_h=1, pad_w=0)),
    (2, 32, 8, 8, dict(out_channels=300, kernel_h=1, kernel_w=1)),
    (5, 1, 28, 28, dict(out_channels=20, kernel_h=5, kernel_w=5)),  # LeNet conv1
    # AlexNet-MoE expert/gating conv1: 24 channels per group (not 16-byte aligned)
    (2, 48, 27, 27, dict(out_channels=64, kernel_h=5, kernel_w=5, pad_h=2, pad_w=2, groups=2)),
    (2, 96, 13, 13, dict(out_channels=64, kernel_h=3, kernel_w=3, pad_h=1, pad_w=1, groups=4)),
]


@pytest.mark.parametrize("case", range(len(CONV_CASES)))
def test_conv_int8_bit_exact(oracle_impl, case):
    N, C, H, W, cp = CONV_CASES[case]
    _conv_case(oracle_impl, np.random.default_rng(100 + case), N, C, H, W, cp, INT8Q)


@pytest.mark.parametrize("dtype", [FP32, FP16])
@pytest.mark.parametrize("case", [0, 1, 2, 5, 8])
def test_conv_float_tolerance(oracle_impl, dtype, case):
    N, C, H, W, cp = CONV_CASES[case]
    _conv_case(oracle_impl, np.random.default_rng(200 + case), N, C, H, W, cp, dtype)


@pytest.mark.parametrize("dims", [(2, 9216, 4096), (3, 4096, 1000), (130, 64, 33), (1, 16, 1)])
def test_inner_product_int8_bit_exact(oracle_impl, dims):
    N, K, O = dims
    rng = np.random.default_rng(300 + K)
    xf = rng.uniform(0, 3, (N, K)).astype(np.float32)
    wf = rng.uniform(-0.05, 0.05, (K, O)).astype(np.float32)
    bias = rng.uniform(-0.2, 0.2, O).astype(np.float32)
    qx, qw = qv_of(oracle_impl, 0, 3), qv_of(oracle_impl, -0.05, 0.05)
    span = 0.1 * np.sqrt(K)
    qo = qv_of(oracle_impl, -span, span)
    x, w = oracle_impl.quantize(xf, qx, INT8Q), oracle_impl.quantize(wf, qw, INT8Q)
    ours = ops.inner_product(x, INT8Q, w, INT8Q, bias, O, qx, qw, qo)
    theirs = oracle_impl.inner_product(x, INT8Q, w, INT8Q, bias, O, qx, qw, qo)
    assert_bits_equal(ours, theirs, f"ip {dims}")


def test_inner_product_float(oracle_impl):
    rng = np.random.default_rng(301)
    x = rng.uniform(-1, 1, (7, 300)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (300, 50)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, 50).astype(np.float32)
    ours = ops.inner_product(x, FP32, w, FP32, b, 50)
    theirs = oracle_impl.inner_product(x, FP32, w, FP32, b, 50)
    assert np.abs(ours - theirs).max() <= 1e-2 * float(theirs.max() - theirs.min())


def test_int8_contraction_depth_bound(oracle_impl):
    """kind::i8 accumulates u8 x u8 products in s32 (the reference in int64,
    src/ops.cpp:73-83): K = 33025 is the deepest exact contraction and still runs
    bit-exact at all-255 operands; K = 33026 is refused with QNB_E_UNSUPPORTED."""
    qx, qw = qv_of(oracle_impl, 0, 3), qv_of(oracle_impl, -0.05, 0.05)
    K = 33025
    x = np.full((2, K), 255, np.uint8)
    w = np.full((K, 16), 255, np.uint8)
    bias = np.zeros(16, np.float32)
    qo = qv_of(oracle_impl, -2000, 2000)
    ours = ops.inner_product(x, INT8Q, w, INT8Q, bias, 16, qx, qw, qo)
    theirs = oracle_impl.inner_product(x, INT8Q, w, INT8Q, bias, 16, qx, qw, qo)
    assert_bits_equal(ours, theirs, "ip K=33025")
    with pytest.raises(ops.QnbError, match="exact s32 accumulation bound") as e:
        ops.inner_product(np.full((2, K + 1), 255, np.uint8), INT8Q, np.full((K + 1, 16), 255, np.uint8), INT8Q,
                          bias, 16, qx, qw, qo)
    assert e.value.status == 10


def test_conv_errors_match_reference():
    x = np.zeros((1, 3, 4, 4), np.float32)
    w = np.zeros((4, 3, 5, 5), np.float32)
    with pytest.raises(ops.QnbError, match="non-positive output extent"):
        ops.conv_forward(x, FP32, w, FP32, None, dict(out_channels=4, kernel_h=5, kernel_w=5))
    with pytest.raises(ops.QnbError, match="group divisibility violation"):
        ops.conv_forward(x, FP32, w, FP32, None, dict(out_channels=4, kernel_h=1, kernel_w=1, groups=2))
    with pytest.raises(ops.QnbError, match="quantized conv requires quantizer values"):
        ops.conv_forward(x.astype(np.uint8), INT8Q, w.astype(np.uint8), INT8Q, None,
                         dict(out_channels=4, kernel_h=1, kernel_w=1))


# ------------------------------------------------------------------- MoE
def test_moe_gate_bit_exact(oracle_impl):
    rng = np.random.default_rng(400)
    B, N, D, K = 256, 16, 16, 4
    feats = rng.normal(0, 4, (B, D)).astype(np.float32)
    wa = rng.uniform(-0.5, 0.5, (N, D)).astype(np.float32)
    for noise in (False, True):
        wb = rng.uniform(-0.2, 0.2, (N, D)).astype(np.float32) if noise else np.zeros((N, D), np.float32)
        wc = rng.uniform(-0.2, 0.2, N).astype(np.float32) if noise else np.zeros(N, np.float32)
        for off in (0, 1000):  # a shard at global sample offset 1000 draws samples 1000..
            idx, w = ops.moe_gate(feats, wa, wb, wc, K, noise, 7, sample_offset=off)
            mism = 0
            for s in range(B):
                _, _, ri, rw = oracle_impl.gating_select(feats[s], wa, wb, wc, K, noise, 7, off + s)
                if not (np.array_equal(idx[s], ri) and np.array_equal(w[s].view(np.uint32), rw.view(np.uint32))):
                    mism += 1
            # the noise table is drawn on the host with the reference's libm arithmetic
            assert mism == 0, (noise, off, mism)


def test_moe_combine_bit_exact():
    from oracle.ffi import Restatement
    rng = np.random.default_rng(401)
    E, B, per, K = 16, 64, 2048, 4
    eo = rng.normal(0, 1, (E, B, per)).astype(np.float32)
    idx = np.stack([rng.permutation(E)[:K] for _ in range(B)]).astype(np.int64)
    w = rng.dirichlet(np.ones(K), B).astype(np.float32)
    assert_bits_equal(ops.moe_combine(eo, idx, w), Restatement().moe_combine(eo, idx, w), "combine")


@pytest.mark.parametrize("npt,ks", [(64, 1), (240, 1), (64, 4), (240, 4), (240, 5)])
def test_inner_product_tiling_and_split_k(oracle_impl, npt, ks, monkeypatch):
    """Wide B tiles (N=256 with the ones row) and split-K (exact s32 partials +
    finalize) must stay bit-exact."""
    monkeypatch.setenv("QNB_IP_NPT", str(npt))
    monkeypatch.setenv("QNB_IP_KSPLIT", str(ks))
    N, K, O = 200, 4096, 1000
    rng = np.random.default_rng(500 + npt + ks)
    xf = rng.uniform(0, 3, (N, K)).astype(np.float32)
    wf = rng.uniform(-0.05, 0.05, (K, O)).astype(np.float32)
    bias = rng.uniform(-0.2, 0.2, O).astype(np.float32)
    qx, qw = qv_of(oracle_impl, 0, 3), qv_of(oracle_impl, -0.05, 0.05)
    span = 0.1 * np.sqrt(K)
    qo = qv_of(oracle_impl, -span, span)
    x, w = oracle_impl.quantize(xf, qx, INT8Q), oracle_impl.quantize(wf, qw, INT8Q)
    ours = ops.inner_product(x, INT8Q, w, INT8Q, bias, O, qx, qw, qo)
    theirs = oracle_impl.inner_product(x, INT8Q, w, INT8Q, bias, O, qx, qw, qo)
    assert_bits_equal(ours, theirs, f"ip npt={npt} ks={ks}")


@pytest.mark.parametrize("mode", ["patch", "cpasync"])
@pytest.mark.parametrize("case", [1, 2, 3, 4])
def test_conv_int8_operand_paths(oracle_impl, case, mode):
    """The alternative A-operand engines (patch planes / plain cp.async gather) are
    bit-exact too; each runs in its own process (the mode switch is read once)."""
    import subprocess, sys, json
    env = dict(os.environ)
    env.pop("QNB_PATCH", None)
    if mode == "patch":
        env["QNB_PATCH"] = "1"
    else:
        env["QNB_NO_TMA"] = "1"
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r); "
        "from test_gpu_ops import _conv_case, CONV_CASES; from oracle import ffi; "
        "o = ffi.Reference() if ffi.have_reference() else ffi.Restatement(); "
        "N, C, H, W, cp = CONV_CASES[%d]; "
        "_conv_case(o, np.random.default_rng(300 + %d), N, C, H, W, cp, 2); print('ok')"
        % (ROOT, os.path.join(ROOT, "tests"), case, case))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
