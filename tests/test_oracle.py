"""Pins the CPU oracle before it is trusted as the checker of the B200 kernels.

1. Known-answer tests taken from the reference's own suites
   (tests/test_quantizer.cpp, test_tensor_core.cpp, test_ops.cpp, test_moe.cpp) and
   the survey-verified extras, run on BOTH the plain-C restatement and
   the compiled reference.
2. Restatement == compiled reference, bit for bit, on seeded random inputs for every
   hot-path function (integer and float islands alike).
"""
import math
import struct

import numpy as np
import pytest

from oracle import ffi

FP32, FP16, INT8Q, INT16Q = 0, 1, 2, 3


def impls():
    out = [ffi.Restatement()]
    if ffi.have_reference():
        out.append(ffi.Reference())
    return out


@pytest.fixture(params=["restatement", "reference"])
def impl(request):
    if request.param == "reference":
        if not ffi.have_reference():
            pytest.skip("oracle/_ref not built")
        return ffi.Reference()
    return ffi.Restatement()


def qv_with_scale(s, zero=0, dtype=INT8Q):
    return ffi.QVals(0.0, 0.0, s, zero, 0.0, 0, 255 if dtype == INT8Q else 65535)


# ------------------------------------------------------------------ KATs
def test_round_half_even_kat(impl):  # tests/test_quantizer.cpp:43-51
    for x, want in [(0.5, 0.0), (1.5, 2.0), (2.5, 2.0), (-0.5, 0.0), (-1.5, -2.0), (3.2, 3.0), (3.7, 4.0)]:
        assert impl.round_half_even(x) == want


def test_estimate_params_kat(impl):  # tests/test_quantizer.cpp:91-111
    qv = impl.estimate_params(0.0, 255.0, INT8Q)
    assert (qv.scale, qv.zero, qv.one, qv.i_min, qv.i_max) == (1.0, 0, 1.0, 0, 255)
    qv = impl.estimate_params(-273.0, 1000.0, INT8Q)
    assert qv.scale == pytest.approx(4.992156862745098, rel=1e-15) and qv.zero == 55
    qv = impl.estimate_params(-394.6, 1832.0, INT8Q)
    assert qv.scale == pytest.approx(8.731764705882354, rel=1e-15) and qv.zero == 45
    with pytest.raises(ffi.OracleError, match="degenerate range"):
        impl.estimate_params(1.0, 1.0, INT8Q)


def test_estimate_from_observation_kat(impl):  # tests/test_quantizer.cpp:134-146
    qv = impl.estimate_from_observation(5.0, 5.0, INT8Q)
    assert qv.f_min == pytest.approx(5.0 - 5.0 / 256.0, rel=1e-12)
    assert qv.f_max == pytest.approx(5.0 + 5.0 / 256.0, rel=1e-12)
    qz = impl.estimate_from_observation(0.0, 0.0, INT8Q)
    assert qz.f_min == pytest.approx(-1.0 / 256.0) and qz.f_max == pytest.approx(1.0 / 256.0)


def test_quantize_kat(impl):  # tests/test_quantizer.cpp:159-168, 181-186
    qv = impl.estimate_params(-273.0, 1000.0, INT8Q)
    assert impl.quantize_value(0.0, qv) == qv.zero
    unit = impl.estimate_params(0.0, 255.0, INT8Q)
    assert impl.quantize_value(3.2, unit) == 3
    assert impl.quantize_value(1e6, unit) == 255
    assert impl.quantize_value(-1e6, unit) == 0
    assert impl.quantize_value(math.inf, unit) == 255
    assert impl.quantize_value(math.nan, unit) == unit.zero
    x = np.array([0.0, 4.992156862745098], np.float32)
    assert list(impl.dequantize(impl.quantize(x, qv, INT8Q), INT8Q, qv)) == pytest.approx(
        [0.0, 4.992156862745098], abs=1e-6)


def test_scale_quant_vals_kat(impl):  # tests/test_quantizer.cpp:265-309
    rq = impl.scale_quant_vals(qv_with_scale(1.0), qv_with_scale(1.0), 31)
    assert (rq.mult, rq.shift, rq.shift_bits) == (1 << 30, -1, 31)
    for x in list(range(0, 1 << 16, 97)) + [65535]:
        assert impl.requant_round(x, rq) == x
    rq = impl.scale_quant_vals(qv_with_scale(1.5), qv_with_scale(1.0), 15)
    assert (rq.mult, rq.shift) == (24576, -1)
    rq = impl.scale_quant_vals(qv_with_scale(2.0), qv_with_scale(3.0), qv_with_scale(4.0), 15)
    assert (rq.mult, rq.shift) == (24576, -1)
    with pytest.raises(ffi.OracleError, match="shift_bits out of range"):
        impl.scale_quant_vals(qv_with_scale(1.0), qv_with_scale(1.0), 0)
    with pytest.raises(ffi.OracleError, match="invalid rescale ratio"):
        impl.scale_quant_vals(qv_with_scale(0.0), qv_with_scale(1.0), 31)


def test_requant_clamp_kat(impl):  # tests/test_quantizer.cpp:330-339
    rq = impl.scale_quant_vals(qv_with_scale(1.0), qv_with_scale(1.0), 31)
    rq.out_zero, rq.out_min, rq.out_max = 10, 0, 255
    assert [impl.requant_clamp(a, rq) for a in (5, 300, -50)] == [15, 255, 0]


def test_requant_ties_to_even_extra(impl):  # SURVEY §8c survey-verified extras
    rq = impl.scale_quant_vals(qv_with_scale(0.5), qv_with_scale(1.0), 31)
    assert [impl.requant_round(a, rq) for a in (-3, -1, 1, 3, 5)] == [-2, 0, 0, 2, 2]


def test_relu_quant_kat(impl):  # tests/test_ops.cpp:80-95 + survey extras (unit ratio, z=128)
    qv = impl.estimate_params(-4.0, 4.0, INT8Q)
    qo = impl.estimate_params(0.0, 4.0, INT8Q)
    rq = impl.scale_quant_vals(qv, qo, 31)
    out = impl.relu_quant(np.array([qv.zero, qv.zero - 5], np.uint8), INT8Q, rq)
    assert list(out) == [qo.zero, qo.zero]
    unit = qv_with_scale(1.0, 128)
    rq = impl.scale_quant_vals(unit, unit, 31)
    out = impl.relu_quant(np.array([129, 130, 131, 229], np.uint8), INT8Q, rq)
    assert list(out) == [128, 130, 130, 228]


def test_fp16_kat(impl):  # tests/test_tensor_core.cpp:68-117
    assert impl.fp16_encode(1.0) == 0x3C00
    assert impl.fp16_encode(0.0) == 0
    assert impl.fp16_encode(65520.0) == 0x7C00
    assert impl.fp16_encode(65504.0) == 0x7BFF
    assert impl.fp16_encode(-2.0) == 0xC000
    assert impl.fp16_decode(0x0001) == math.ldexp(1.0, -24)
    assert impl.fp16_decode(0xFC00) == -math.inf
    assert impl.fp16_encode(6.1035156e-5) == 0x0400
    assert impl.fp16_encode(6.0975552e-5) == 0x03FF


def test_fp16_round_trip_all_patterns(restatement):  # tests/test_tensor_core.cpp:88-99
    pats = np.arange(65536, dtype=np.uint16)
    dec = restatement.cast_float(pats, FP16, FP32)
    keep = ~np.isnan(dec)
    assert keep.sum() == 65536 - 2046
    enc = restatement.cast_float(dec[keep], FP32, FP16)
    assert np.array_equal(enc, pats[keep])


def test_pool_kat(impl):  # tests/test_ops.cpp:451-465
    out = impl.pool_max(np.full((1, 1, 4, 4), 3.5, np.float32), FP32, 2, 2)
    assert out.shape == (1, 1, 2, 2) and np.all(out == 3.5)
    out = impl.pool_max(np.array([1, 2, 3, 4], np.float32).reshape(1, 1, 2, 2), FP32, 2, 2)
    assert out.reshape(-1).tolist() == [4.0]


def test_select_topk_kat(impl):  # tests/test_moe.cpp:166-194 (through the gating path)
    # p from a hand-picked logit vector: log of the target probabilities.
    p = np.array([0.1, 0.4, 0.3, 0.2], np.float32)
    wa = np.eye(4, dtype=np.float32)
    x = np.log(p).astype(np.float32)
    _, pp, idx, w = impl.gating_select(x, wa, np.zeros_like(wa), np.zeros(4, np.float32), 2)
    assert list(idx) == [1, 2]
    assert w[0] == pytest.approx(0.4 / 0.7, rel=1e-6) and w[1] == pytest.approx(0.3 / 0.7, rel=1e-6)
    x = np.zeros(4, np.float32)
    _, _, idx, _ = impl.gating_select(x, wa, np.zeros_like(wa), np.zeros(4, np.float32), 2)
    assert list(idx) == [0, 1]  # ties toward the lower index


def test_quantized_conv_hand_case(impl):
    # 1x1x3x3 input, 2x2 kernel of ones, identity grids: dot products are window sums.
    qv = ffi.QVals(0.0, 255.0, 1.0, 0, 1.0, 0, 255)
    x = np.arange(1, 10, dtype=np.uint8).reshape(1, 1, 3, 3)
    w = np.ones((1, 1, 2, 2), np.uint8)
    out = impl.conv_forward(x, INT8Q, w, INT8Q, None, dict(out_channels=1, kernel_h=2, kernel_w=2), qv, qv, qv)
    assert out.reshape(-1).tolist() == [12, 16, 24, 28]


# ------------------------------------------- restatement == reference (random)
needs_ref = pytest.mark.skipif(not ffi.have_reference(), reason="oracle/_ref not built")


def rand_qv(rng, dtype):
    lo = rng.uniform(-5, 0.5)
    return ffi.Restatement().estimate_params(lo, lo + rng.uniform(0.1, 10), dtype)


@needs_ref
@pytest.mark.parametrize("dtype", [INT8Q, INT16Q])
def test_parity_quantize_dequantize(restatement, reference, dtype):
    rng = np.random.default_rng(1)
    qv = rand_qv(rng, dtype)
    x = rng.uniform(-20, 20, 5000).astype(np.float32)
    x[:4] = [np.nan, np.inf, -np.inf, 0.0]
    a, b = restatement.quantize(x, qv, dtype), reference.quantize(x, qv, dtype)
    assert np.array_equal(a, b)
    assert np.array_equal(restatement.dequantize(a, dtype, qv).view(np.uint32),
                          reference.dequantize(a, dtype, qv).view(np.uint32))


@needs_ref
def test_parity_requant_random(restatement, reference):
    rng = np.random.default_rng(2)
    for trial in range(300):
        dt = INT8Q if trial % 2 else INT16Q
        qa, qb, qc = (rand_qv(rng, dt) for _ in range(3))
        sb = int(rng.integers(1, 32))
        r1 = restatement.scale_quant_vals(qa, qb, qc, sb)
        r2 = reference.scale_quant_vals(qa, qb, qc, sb)
        assert r1.as_tuple() == r2.as_tuple()
        u1 = restatement.scale_quant_vals(qa, qc, sb)
        assert u1.as_tuple() == reference.scale_quant_vals(qa, qc, sb).as_tuple()
        for acc in rng.integers(-(1 << 40), 1 << 40, 20):
            assert restatement.requant_clamp(int(acc), r1) == reference.requant_clamp(int(acc), r2)
        q = rng.integers(0, 256 if dt == INT8Q else 65536, 64).astype(np.uint8 if dt == INT8Q else np.uint16)
        assert np.array_equal(restatement.relu_quant(q, dt, u1), reference.relu_quant(q, dt, u1))


@needs_ref
@pytest.mark.parametrize("dtype", [INT8Q, FP32, FP16])
@pytest.mark.parametrize("geom", [
    dict(C=3, H=23, W=23, out_channels=8, kernel_h=11, kernel_w=11, stride_h=4, stride_w=4),   # conv1-like
    dict(C=8, H=9, W=9, out_channels=6, kernel_h=5, kernel_w=5, pad_h=2, pad_w=2, groups=2),   # conv2-like
    dict(C=6, H=7, W=6, out_channels=4, kernel_h=3, kernel_w=3, pad_h=1, pad_w=1, stride_h=2),
])
def test_parity_conv(restatement, reference, dtype, geom):
    rng = np.random.default_rng(3)
    g = dict(geom)
    C_, H, W = g.pop("C"), g.pop("H"), g.pop("W")
    cp = dict(g)
    G = cp.get("groups", 1)
    xf = rng.uniform(-2, 2, (2, C_, H, W)).astype(np.float32)
    wf = rng.uniform(-0.5, 0.5, (cp["out_channels"], C_ // G, cp["kernel_h"], cp["kernel_w"])).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, cp["out_channels"]).astype(np.float32)
    if dtype == INT8Q:
        qx, qw, qo = (restatement.estimate_params(-2, 2, INT8Q), restatement.estimate_params(-0.5, 0.5, INT8Q),
                      restatement.estimate_params(-3, 4, INT8Q))
        x, w = restatement.quantize(xf, qx, INT8Q), restatement.quantize(wf, qw, INT8Q)
        a = restatement.conv_forward(x, dtype, w, dtype, bias, cp, qx, qw, qo)
        b = reference.conv_forward(x, dtype, w, dtype, bias, cp, qx, qw, qo)
    else:
        x = xf if dtype == FP32 else restatement.cast_float(xf, FP32, FP16)
        a = restatement.conv_forward(x, dtype, wf, FP32, bias, cp)
        b = reference.conv_forward(x, dtype, wf, FP32, bias, cp)
    assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@needs_ref
@pytest.mark.parametrize("dtype", [INT8Q, INT16Q, FP32])
def test_parity_inner_product(restatement, reference, dtype):
    rng = np.random.default_rng(4)
    xf = rng.uniform(-1, 1, (5, 37)).astype(np.float32)
    wf = rng.uniform(-0.3, 0.3, (37, 11)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, 11).astype(np.float32)
    if dtype == FP32:
        a = restatement.inner_product(xf, dtype, wf, FP32, bias, 11)
        b = reference.inner_product(xf, dtype, wf, FP32, bias, 11)
    else:
        qx, qw, qo = (restatement.estimate_params(-1, 1, dtype), restatement.estimate_params(-0.3, 0.3, dtype),
                      restatement.estimate_params(-2, 2, dtype))
        x, w = restatement.quantize(xf, qx, dtype), restatement.quantize(wf, qw, dtype)
        a = restatement.inner_product(x, dtype, w, dtype, bias, 11, qx, qw, qo)
        b = reference.inner_product(x, dtype, w, dtype, bias, 11, qx, qw, qo)
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


@needs_ref
def test_parity_float_islands(restatement, reference):
    rng = np.random.default_rng(5)
    x = rng.uniform(-30, 60, (3, 12, 5, 4)).astype(np.float32)
    assert np.array_equal(restatement.lrn(x).view(np.uint32), reference.lrn(x).view(np.uint32))
    s = rng.normal(0, 5, (4, 1000)).astype(np.float32)
    assert np.array_equal(restatement.softmax(s).view(np.uint32), reference.softmax(s).view(np.uint32))
    for dt in (INT8Q, FP32, FP16):
        xi = x if dt == FP32 else (restatement.cast_float(x, FP32, FP16) if dt == FP16
                                   else rng.integers(0, 256, x.shape).astype(np.uint8))
        assert np.array_equal(restatement.pool_max(xi, dt, 3, 2).view(np.uint8),
                              reference.pool_max(xi, dt, 3, 2).view(np.uint8))
    y = rng.uniform(-3, 3, 999).astype(np.float32)
    y16 = restatement.cast_float(y, FP32, FP16)
    assert np.array_equal(y16, reference.cast_float(y, FP32, FP16))
    assert np.array_equal(restatement.relu_float(y, FP32, 0.0).view(np.uint32),
                          reference.relu_float(y, FP32, 0.0).view(np.uint32))


@needs_ref
def test_parity_gating(restatement, reference):
    rng = np.random.default_rng(6)
    for trial in range(50):
        N, D = 16, 16
        x = rng.normal(0, 3, D).astype(np.float32)
        wa = rng.uniform(-0.5, 0.5, (N, D)).astype(np.float32)
        wb = rng.uniform(-0.2, 0.2, (N, D)).astype(np.float32)
        wc = rng.uniform(-0.2, 0.2, N).astype(np.float32)
        noise = trial % 2 == 1
        a = restatement.gating_select(x, wa, wb, wc, 4, noise, 99, trial)
        b = reference.gating_select(x, wa, wb, wc, 4, noise, 99, trial)
        for u, v in zip(a, b):
            assert np.array_equal(u.view(np.uint8), v.view(np.uint8))


@needs_ref
def test_moe_combine_matches_reference_moe_forward(restatement, reference):
    # PER_SAMPLE and ALL_EXPERTS are bit-identical (tests/test_moe.cpp:264-317); the
    # restated combine must match both.
    rng = np.random.default_rng(7)
    B, N, D, per, K = 12, 8, 6, 10, 3
    feats = rng.normal(0, 2, (B, D)).astype(np.float32)
    wa = rng.uniform(-0.5, 0.5, (N, D)).astype(np.float32)
    wb, wc = np.zeros_like(wa), np.zeros(N, np.float32)
    eo = rng.normal(0, 1, (N, B, per)).astype(np.float32)
    inp = np.arange(B, dtype=np.float32).reshape(B, 1)  # carries the sample index
    idx = np.empty((B, K), np.int64)
    w = np.empty((B, K), np.float32)
    for s in range(B):
        _, _, idx[s], w[s] = restatement.gating_select(feats[s], wa, wb, wc, K, False, 0, s)
    ours = restatement.moe_combine(eo, idx, w)
    for mode in (0, 1):
        theirs = reference.moe_forward_fixed(inp, feats, wa, wb, wc, K, eo, mode=mode)
        assert np.array_equal(ours.view(np.uint32), theirs.view(np.uint32))


def test_glibc_expf_restatement_matches_libm():
    """qnb_gating_expf restates glibc's expf; check it against this host's libm."""
    from paper_2209_15427_b200 import ops
    import ctypes
    libm = ctypes.CDLL("libm.so.6")
    libm.expf.restype = ctypes.c_float
    libm.expf.argtypes = [ctypes.c_float]
    rng = np.random.default_rng(8)
    xs = np.concatenate([rng.uniform(-104, 89, 20000), rng.normal(0, 3, 20000)]).astype(np.float32)
    for x in xs:
        a, b = ops.gating_expf(float(x)), libm.expf(float(x))
        assert struct.pack("f", a) == struct.pack("f", b), x


def test_host_gating_noise_matches_reference(reference):
    """qnb_gating_noise (the table the device gate reads) is the reference's
    gating_noise bit for bit (src/moe.cpp:53-71) over many (seed, sample, expert, stream)."""
    from paper_2209_15427_b200 import ops
    rng = np.random.default_rng(9)
    for seed in (0, 7, 99, 2**63 + 5):
        for sample in list(range(40)) + [int(v) for v in rng.integers(0, 1 << 40, 40)]:
            for expert in (0, 3, 15):
                for stream in (0, 1):
                    a = ops.gating_noise(seed, sample, expert, stream)
                    b = reference.gating_noise(seed, sample, expert, stream)
                    assert struct.pack("f", a) == struct.pack("f", b), (seed, sample, expert, stream)
