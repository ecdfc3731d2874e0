"""Debug: dump the first patch tile's A planes and B stage 0, compare with expectations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import ffi
from paper_2209_15427_b200 import ops
from paper_2209_15427_b200._lib import INT8Q
os.environ["QNB_PATCH_DUMP"] = "/tmp/patch_dump.bin"
o = ffi.Restatement()
rng = np.random.default_rng(0)
C, H, K, pad, OC = 32, 13, 3, 1, 64
qx, qw, qo = (o.estimate_params(-2, 2.5, INT8Q), o.estimate_params(-0.5, 0.55, INT8Q), o.estimate_params(-8, 9, INT8Q))
x = o.quantize(rng.uniform(-2, 2, (1, C, H, H)).astype(np.float32), qx, INT8Q)
w = o.quantize(rng.uniform(-0.5, 0.5, (OC, C, K, K)).astype(np.float32), qw, INT8Q)
cp = dict(out_channels=OC, kernel_h=K, kernel_w=K, pad_h=pad, pad_w=pad)
ours = ops.conv_forward(x, INT8Q, w, INT8Q, np.zeros(OC, np.float32), cp, qx, qw, qo)
theirs = o.conv_forward(x, INT8Q, w, INT8Q, np.zeros(OC, np.float32), cp, qx, qw, qo)
print("conv mismatches", int((ours != theirs).sum()), "of", ours.size)
d = np.fromfile("/tmp/patch_dump.bin", np.uint8)
wp = H + 2 * pad
R = (wp + 125 + K) // wp + K
plane = ((R * wp * 16 + 127) // 128) * 128 + 64
xp = np.full((wp, wp, C), qx.zero, np.uint8); xp[pad:pad + H, pad:pad + H] = x[0].transpose(1, 2, 0)
for b in range(2):
    got = d[b * plane: b * plane + R * wp * 16].reshape(R * wp, 16)
    exp = np.zeros((R * wp, 16), np.uint8)
    for q in range(R * wp):
        y = min(q // wp, wp - 1); xx = q % wp
        exp[q] = xp[y, xx, b * 16:(b + 1) * 16]
    bad = np.argwhere(got != exp)
    print("plane", b, "mismatch", len(bad), bad[:5].tolist(), got[:2].tolist(), exp[:2].tolist())
nrows = ((OC + 1 + 15) // 16) * 16
B = d[2 * plane:2 * plane + nrows * 128]
Bm = B.reshape(nrows, 128)
# unswizzle SW128
un = np.zeros_like(Bm)
for r in range(nrows):
    for ch in range(8):
        un[r, ch * 16:(ch + 1) * 16] = Bm[r, ((ch ^ (r & 7)) * 16):((ch ^ (r & 7)) * 16 + 16)]
# expected B stage 0: K steps 0..3 = taps (0,0),(0,1),(0,2),(1,0) of pair 0: bytes 0-15 block0 ch 0-15, 16-31 block1 ch 16-31
taps = [(0, 0), (0, 1), (0, 2), (1, 0)]
exp = np.zeros((OC, 128), np.uint8)
for q, (r, s) in enumerate(taps):
    for e in range(32):
        exp[:, q * 32 + e] = w[:, e, r, s]
print("B mismatch", int((un[:OC] != exp).sum()), "ones row", un[OC][:40].tolist())
# raw accumulators of tile 0 vs. the GEMM of the whole tile computed on the host
nr = nrows
acc = d[2 * plane + nr * 128:2 * plane + nr * 128 + 128 * nr * 4].view(np.int32).reshape(128, nr)
# host: for each grid pixel m (tile 0: P = m), sum over taps/channels of xp * w (raw u8 products) and rowsum
want = np.zeros((128, OC), np.int64); rows = np.zeros(128, np.int64)
for m in range(128):
    Y, X = m // wp, m % wp
    for r in range(K):
        for s_ in range(K):
            yy, xx = Y + r, X + s_
            if yy >= wp: yy = wp - 1
            px = xp[yy, xx] if xx < wp else xp[yy + 1 if yy + 1 < wp else yy, xx - wp]
            want[m] += (w[:, :, r, s_].astype(np.int64) * px[None, :].astype(np.int64)).sum(1)
            rows[m] += px.astype(np.int64).sum()
print("acc mismatch", int((acc[:, :OC] != want).sum()), "rowsum mismatch", int((acc[:, OC] != rows).sum()))
for m in [0, 1, 15, 16, 17]:
    print(m, acc[m, :4].tolist(), want[m, :4].tolist(), acc[m, OC], rows[m])
for m in [0, 1, 15, 16, 17, 40]:
    Y, X = m // wp, m % wp
    contrib = {}
    for r in range(K):
        for s_ in range(K):
            q = (Y + r) * wp + X + s_
            yy, xx = min(q // wp, wp - 1), q % wp
            contrib[(r, s_)] = int(xp[yy, xx].astype(np.int64).sum())
    deficit = int(rows[m] - acc[m, OC])
    print(m, "deficit", deficit, "taps matching", [t for t, v in contrib.items() if v == deficit], contrib)
