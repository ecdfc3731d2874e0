"""Checkpoint-by-checkpoint FP16 AlexNet comparison (diagnostic detail for the
float-network tolerance test)."""
import json

import numpy as np
import pytest

from oracle import ffi
from paper_2209_15427_b200 import graph as G
from paper_2209_15427_b200 import graphs
from paper_2209_15427_b200.net import Net

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision,batch", [("fp16", 2)])
def test_alexnet_float_checkpoints(precision, batch):
    if not ffi.have_reference():
        pytest.skip("needs oracle/_ref")
    ref = ffi.Reference()
    g = graphs.alexnet(1)
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    params = graphs.synth_params(g, shapes)
    x = graphs.synth_images(batch, (3, 227, 227), offset=7)
    names = [l["name"] for l in g["layers"]]
    report = []
    for ck in ("conv1", "relu1", "pool1", "norm1", "conv2", "relu5", "pool5", "fc6", "relu7", "fc8"):
        prefix = {"name": "p", "layers": g["layers"][: names.index(ck) + 1]}
        pr = {k: v for k, v in params.items() if k.split(".")[0] in names[: names.index(ck) + 1]}
        ours = Net(G.override_precision(prefix, precision) if precision != "fp32" else prefix)
        for k, v in pr.items():
            ours.set_param(k, v)
        mine = list(ours.forward({"data": x}).values())[0]
        rn = ref.net(json.dumps(prefix), 1 if precision == "fp16" else -1)
        for k, v in pr.items():
            rn.set_param(k, v)
        rn.set_mode(3)  # typed execution
        (arr, dt, _), = rn.forward("data", x).values()
        R = ffi.Restatement()
        a = R.cast_float(mine, 1, 0) if mine.dtype == np.uint16 else mine
        b = R.cast_float(arr, 1, 0) if dt == 1 else arr
        rng = float(b.max() - b.min())
        err = float(np.abs(a.astype(np.float64) - b).max())
        report.append((ck, err, rng, a.reshape(-1)[:3].tolist(), b.reshape(-1)[:3].tolist()))
    for r in report:
        print(precision, batch, r)
    bad = [r for r in report if not (r[1] <= 1e-2 * r[2])]
    assert not bad, bad
