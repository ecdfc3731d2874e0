"""Debug probe for the patch-mode conv: single-tap weights, compare with the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import ffi
from paper_2209_15427_b200 import ops
from paper_2209_15427_b200._lib import INT8Q
o = ffi.Reference() if ffi.have_reference() else ffi.Restatement()
rng = np.random.default_rng(0)
def qv(lo, hi): return o.estimate_params(lo, hi, INT8Q)
for (C, H, K, G, pad) in [(32, 13, 3, 1, 1), (256, 13, 3, 1, 1), (96, 27, 5, 2, 2)]:
    cp = dict(out_channels=64 * G, kernel_h=K, kernel_w=K, pad_h=pad, pad_w=pad, groups=G)
    qx, qw, qo = qv(-2, 2.5), qv(-0.5, 0.55), qv(-8, 9)
    x = o.quantize(rng.uniform(-2, 2, (1, C, H, H)).astype(np.float32), qx, INT8Q)
    for tap in [(0, 0), (0, 1), (1, 0), (1, 1), None]:
        wf = rng.uniform(-0.5, 0.5, (64 * G, C // G, K, K)).astype(np.float32)
        if tap is not None:
            m = np.zeros_like(wf); m[:, :, tap[0], tap[1]] = 1; wf = wf * m
        w = o.quantize(wf, qw, INT8Q)
        if tap is not None:  # zero-point weights elsewhere (w - zw = 0)
            zw = qw.zero
            w2 = np.full_like(w, zw); w2[:, :, tap[0], tap[1]] = w[:, :, tap[0], tap[1]]; w = w2
        b = np.zeros(64 * G, np.float32)
        ours = ops.conv_forward(x, INT8Q, w, INT8Q, b, cp, qx, qw, qo)
        theirs = o.conv_forward(x, INT8Q, w, INT8Q, b, cp, qx, qw, qo)
        bad = np.argwhere(ours != theirs)
        print(C, H, K, G, "tap", tap, "mismatch", len(bad), "of", ours.size, bad[:4].tolist(), flush=True)
