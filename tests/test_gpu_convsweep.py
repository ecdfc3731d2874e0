"""Parity at the single conv-layer sweep shapes (BASELINE configs[4]; bench.py --model
convsweep): the compiled plan for one convolution (C = K, R x R, stride s, pad R // 2) vs
the UNMODIFIED reference Net on the same seeded weights, grids and images.  INT8 byte-exact,
FP16 within 1e-2 x output range (north_star).  Spatial sizes are reduced from 56x56 so the
reference finishes in seconds; the engine choice depends on channels, filter and stride,
which are the sweep's."""
import json

import numpy as np
import pytest

from oracle import ffi
from paper_2209_15427_b200 import graph as G
from paper_2209_15427_b200 import graphs
from paper_2209_15427_b200.net import QUANTIZED, Net

pytestmark = pytest.mark.gpu
DT = {"fp32": 0, "fp16": 1, "int8": 2, "int16": 3}

CASES = [  # (C = K, R, stride, input resolution)
    (64, 11, 4, 56), (64, 3, 1, 28), (128, 5, 2, 28), (256, 3, 1, 20), (256, 11, 2, 24),
    (512, 3, 2, 20), (512, 5, 1, 12),
]


def run(case, precision):
    if not ffi.have_reference():
        pytest.skip("needs oracle/_ref")
    C, R, S, res = case
    N = 2
    g = graphs.conv_layer(N, C, res, C, R, S)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    params = graphs.synth_params(g, shapes)
    ranges = {"data": (0.0, 255.0), "conv": (-150.0, 150.0)}
    x = graphs.synth_images(N, (C, res, res), offset=31)
    ours = Net(G.override_precision(g, precision))
    for k, v in params.items():
        ours.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        ours.set_range(k, lo, hi)
    ours.finalize_quantizers()
    ours.set_quant_mode(QUANTIZED)
    mine = ours.forward({"data": x})["conv"]
    ref = ffi.Reference().net(json.dumps(g), DT[precision])
    for k, v in params.items():
        ref.set_param(k, v)
    for k, (lo, hi) in ranges.items():
        ref.set_range(k, lo, hi)
    ref.finalize()
    ref.set_mode(3)
    (theirs, dt, qv), = ref.forward("data", x).values()
    return mine, theirs


@pytest.mark.parametrize("case", CASES)
def test_convsweep_int8_bit_exact(case):
    mine, theirs = run(case, "int8")
    assert mine.dtype == theirs.dtype and mine.shape == theirs.shape
    mism = int((mine != theirs).sum())
    assert mism == 0, f"{case}: {mism} of {theirs.size} differ"
    assert len(np.unique(theirs)) > 16


@pytest.mark.parametrize("case", [CASES[0], CASES[2], CASES[3], CASES[6]])
def test_convsweep_fp16_within_tolerance(case):
    mine, theirs = run(case, "fp16")
    r = ffi.Restatement()
    a = r.cast_float(mine, 1, 0)  # FP16 bits -> FP32
    b = r.cast_float(theirs, 1, 0)
    err = float(np.abs(a.astype(np.float64) - b).max())
    rng = float(b.max() - b.min())
    assert err <= 1e-2 * rng, (case, err, rng)
