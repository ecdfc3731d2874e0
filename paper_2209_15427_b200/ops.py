"""Host-side mirror of the reference operator API over the qnb C-ABI.

Each function has the name and argument meaning of the reference free function it
replaces (include/qnet/{ops,quantizer,moe}.hpp) and raises QnbError carrying the
reference's message for the reference's error cases.  Tensors are numpy arrays in
the reference's own layout (dense row-major NCHW); quantized tensors are uint8
(INT8Q) or uint16 (INT16Q) arrays whose QuantizerValues are passed explicitly.
Every call moves data to the B200, runs the sm_100a kernel and copies back — this
is the parity surface; the throughput path is the compiled plan (plan.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from ._lib import FP16, FP32, INT8Q, INT16Q, ConvParams, QnbError, QVals, Requant, check

NP_OF = {FP32: np.float32, FP16: np.uint16, INT8Q: np.uint8, INT16Q: np.uint16}


class DeviceArray:
    """A device allocation owned by Python (qnb_malloc / qnb_free)."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        self.ptr = C.c_void_p()
        check(L.lib().qnb_malloc(C.byref(self.ptr), max(self.nbytes, 1)))

    @classmethod
    def from_numpy(cls, a: np.ndarray) -> "DeviceArray":
        a = np.ascontiguousarray(a)
        d = cls(a.nbytes)
        if a.nbytes:
            check(L.lib().qnb_memcpy_h2d(d.ptr, a.ctypes.data_as(C.c_void_p), a.nbytes, None))
        return d

    def to_numpy(self, dtype, shape) -> np.ndarray:
        out = np.empty(shape, dtype=dtype)
        if out.nbytes:
            check(L.lib().qnb_memcpy_d2h(out.ctypes.data_as(C.c_void_p), self.ptr, out.nbytes, None))
            check(L.lib().qnb_stream_sync(None))
        return out

    def __del__(self):
        try:
            if self.ptr:
                L.lib().qnb_free(self.ptr)
                self.ptr = C.c_void_p()
        except Exception:
            pass


def _qv(qv) -> QVals:
    if qv is None or isinstance(qv, QVals):
        return qv
    if hasattr(qv, "as_tuple"):
        return QVals(*qv.as_tuple())
    return QVals(*qv)


def _rq(rq) -> Requant:
    if isinstance(rq, Requant):
        return rq
    if hasattr(rq, "as_tuple"):
        return Requant(*rq.as_tuple())
    return Requant(*rq)


def _ref(x):
    return C.byref(x) if x is not None else None


# ------------------------------------------------------------ quantizer math
def round_half_even(x: float) -> float:
    return L.lib().qnb_round_half_even(float(x))


def estimate_params(f_min: float, f_max: float, dtype: int) -> QVals:
    out = QVals()
    check(L.lib().qnb_estimate_params(f_min, f_max, dtype, C.byref(out)))
    return out


def estimate_from_observation(seen_min: float, seen_max: float, dtype: int) -> QVals:
    out = QVals()
    check(L.lib().qnb_estimate_from_observation(seen_min, seen_max, dtype, C.byref(out)))
    return out


def scale_quant_vals(*args) -> Requant:
    """scale_quant_vals(qv_in, qv_out, sb) or scale_quant_vals(qv_a, qv_b, qv_c, sb)."""
    rq = Requant()
    if len(args) == 3:
        check(L.lib().qnb_scale_quant_vals(_ref(_qv(args[0])), _ref(_qv(args[1])), int(args[2]), C.byref(rq)))
    else:
        check(L.lib().qnb_scale_quant_vals3(_ref(_qv(args[0])), _ref(_qv(args[1])), _ref(_qv(args[2])),
                                            int(args[3]), C.byref(rq)))
    return rq


def requant_clamp(acc: int, rq: Requant) -> int:
    return L.lib().qnb_requant_clamp_host(int(acc), C.byref(_rq(rq)))


# ------------------------------------------------------------------ ops
def quantize(x: np.ndarray, qv, dtype: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    dx = DeviceArray.from_numpy(x)
    dy = DeviceArray(x.size * (1 if dtype == INT8Q else 2))
    check(L.lib().qnb_quantize(dx.ptr, x.size, _ref(_qv(qv)), dtype, dy.ptr, None))
    return dy.to_numpy(NP_OF[dtype], x.shape)


def dequantize(q: np.ndarray, dtype: int, qv) -> np.ndarray:
    dq = DeviceArray.from_numpy(q)
    dy = DeviceArray(q.size * 4)
    check(L.lib().qnb_dequantize(dq.ptr, q.size, dtype, _ref(_qv(qv)), dy.ptr, None))
    return dy.to_numpy(np.float32, q.shape)


def requantize(q: np.ndarray, in_dtype: int, rq: Requant, out_dtype: int) -> np.ndarray:
    """The int -> int QUANTIZER layer (src/net.cpp:483-493)."""
    dq = DeviceArray.from_numpy(q)
    dy = DeviceArray(q.size * (1 if out_dtype == INT8Q else 2))
    check(L.lib().qnb_requantize(dq.ptr, q.size, in_dtype, C.byref(_rq(rq)), out_dtype, dy.ptr, None))
    return dy.to_numpy(NP_OF[out_dtype], q.shape)


def relu_quant(q: np.ndarray, dtype: int, rq: Requant) -> np.ndarray:
    dq = DeviceArray.from_numpy(q)
    dy = DeviceArray(q.nbytes)
    check(L.lib().qnb_relu_quant(dq.ptr, q.size, dtype, C.byref(_rq(rq)), dy.ptr, None))
    return dy.to_numpy(q.dtype, q.shape)


def relu_float(x: np.ndarray, dtype: int, negative_slope: float) -> np.ndarray:
    dx = DeviceArray.from_numpy(x)
    dy = DeviceArray(x.nbytes)
    check(L.lib().qnb_relu_float(dx.ptr, x.size, dtype, C.c_float(negative_slope), dy.ptr, None))
    return dy.to_numpy(x.dtype, x.shape)


def cast_float(x: np.ndarray, from_dtype: int, to_dtype: int) -> np.ndarray:
    dx = DeviceArray.from_numpy(x)
    dy = DeviceArray(x.size * (4 if to_dtype == FP32 else 2))
    check(L.lib().qnb_cast_float(dx.ptr, x.size, from_dtype, to_dtype, dy.ptr, None))
    return dy.to_numpy(NP_OF[to_dtype], x.shape)


def pool_max(x: np.ndarray, dtype: int, kernel: int, stride: int) -> np.ndarray:
    N, Ch, H, W = x.shape
    oh, ow = (H - kernel) // stride + 1, (W - kernel) // stride + 1
    shape = (C.c_int64 * 4)(N, Ch, H, W)
    dx = DeviceArray.from_numpy(x)
    dy = DeviceArray(max(N * Ch * max(oh, 0) * max(ow, 0), 0) * x.itemsize)
    check(L.lib().qnb_pool_max(dx.ptr, shape, dtype, kernel, stride, dy.ptr, None))
    return dy.to_numpy(x.dtype, (N, Ch, oh, ow))


def lrn(x: np.ndarray, local_size=5, alpha=1e-4, beta=0.75, k=1.0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    N, Ch = x.shape[0], x.shape[1]
    S = x.size // max(N * Ch, 1)
    dx = DeviceArray.from_numpy(x)
    dy = DeviceArray(x.nbytes)
    check(L.lib().qnb_lrn(dx.ptr, N, Ch, S, local_size, alpha, beta, k, dy.ptr, None))
    return dy.to_numpy(np.float32, x.shape)


def softmax(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    N = x.shape[0]
    F = x.size // max(N, 1)
    dx = DeviceArray.from_numpy(x)
    dy = DeviceArray(x.nbytes)
    check(L.lib().qnb_softmax(dx.ptr, N, F, dy.ptr, None))
    return dy.to_numpy(np.float32, x.shape)


def conv_forward(x: np.ndarray, dtype: int, weight: np.ndarray, w_dtype: int, bias, cp: dict,
                 in_qv=None, w_qv=None, out_qv=None, shift_bits: int = 0) -> np.ndarray:
    """qnet::conv_forward (src/ops.cpp:264-342) on the B200."""
    p = ConvParams(cp["out_channels"], cp.get("kernel_h", 1), cp.get("kernel_w", 1), cp.get("stride_h", 1),
                   cp.get("stride_w", 1), cp.get("pad_h", 0), cp.get("pad_w", 0), cp.get("groups", 1),
                   1 if bias is not None else 0)
    xs = (C.c_int64 * 4)(*x.shape)
    ys = (C.c_int64 * 4)()
    dx = DeviceArray.from_numpy(x)
    dw = DeviceArray.from_numpy(weight)
    db = DeviceArray.from_numpy(np.ascontiguousarray(bias, dtype=np.float32)) if bias is not None else None
    N, Ch, H, W = x.shape
    oh = (H + 2 * p.pad_h - p.kernel_h) // p.stride_h + 1
    ow = (W + 2 * p.pad_w - p.kernel_w) // p.stride_w + 1
    out_es = {FP32: 4, FP16: 2, INT8Q: 1, INT16Q: 2}[dtype]
    dy = DeviceArray(max(N * p.out_channels * max(oh, 1) * max(ow, 1) * out_es, 1))
    check(L.lib().qnb_conv_forward(dx.ptr, xs, dtype, _ref(_qv(in_qv)), dw.ptr, w_dtype, _ref(_qv(w_qv)),
                                   db.ptr if db is not None else None, C.byref(p), _ref(_qv(out_qv)),
                                   shift_bits, dy.ptr, ys, None))
    return dy.to_numpy(NP_OF[dtype], tuple(ys))


def inner_product(x: np.ndarray, dtype: int, weight: np.ndarray, w_dtype: int, bias, out_features: int,
                  in_qv=None, w_qv=None, out_qv=None, shift_bits: int = 0) -> np.ndarray:
    """qnet::inner_product (src/ops.cpp:392-443): x flattened to N x K, weight K x out."""
    N = x.shape[0]
    K = x.size // max(N, 1)
    dx = DeviceArray.from_numpy(x)
    dw = DeviceArray.from_numpy(weight)
    db = DeviceArray.from_numpy(np.ascontiguousarray(bias, dtype=np.float32)) if bias is not None else None
    out_es = {FP32: 4, FP16: 2, INT8Q: 1, INT16Q: 2}[dtype]
    dy = DeviceArray(max(N * out_features * out_es, 1))
    check(L.lib().qnb_inner_product(dx.ptr, N, K, dtype, _ref(_qv(in_qv)), dw.ptr, w_dtype, _ref(_qv(w_qv)),
                                    db.ptr if db is not None else None, out_features, _ref(_qv(out_qv)),
                                    shift_bits, dy.ptr, None))
    return dy.to_numpy(NP_OF[dtype], (N, out_features))


def gating_noise(seed: int, sample: int, expert: int, stream: int) -> float:
    """gating_noise (src/moe.cpp:53-71), host restatement used for the device table."""
    return float(L.lib().qnb_gating_noise(seed, sample, expert, stream))


def moe_gate(feats: np.ndarray, wa: np.ndarray, wb: np.ndarray, wc: np.ndarray, top_k: int,
             noise_enabled: bool = False, seed: int = 0, sample_offset: int = 0):
    """gating_logits + gating_probs + select_topk per sample (src/moe.cpp:73-144)."""
    B, D = feats.shape
    N = wa.shape[0]
    bufs = [DeviceArray.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) for a in (feats, wa, wb, wc)]
    didx = DeviceArray(B * top_k * 8)
    dw = DeviceArray(B * top_k * 4)
    check(L.lib().qnb_moe_gate_at(bufs[0].ptr, B, D, bufs[1].ptr, bufs[2].ptr, bufs[3].ptr, N, top_k,
                                  1 if noise_enabled else 0, seed, sample_offset, didx.ptr, dw.ptr, None))
    return didx.to_numpy(np.int64, (B, top_k)), dw.to_numpy(np.float32, (B, top_k))


def moe_combine(expert_out: np.ndarray, idx: np.ndarray, weights: np.ndarray) -> np.ndarray:
    """Weighted combine in selection order; expert_out is [n_experts][B][per]."""
    E, B, per = expert_out.shape
    K = idx.shape[1]
    de = DeviceArray.from_numpy(np.ascontiguousarray(expert_out, dtype=np.float32))
    di = DeviceArray.from_numpy(np.ascontiguousarray(idx, dtype=np.int64))
    dw = DeviceArray.from_numpy(np.ascontiguousarray(weights, dtype=np.float32))
    dy = DeviceArray(B * per * 4)
    check(L.lib().qnb_moe_combine(de.ptr, B, per, K, di.ptr, dw.ptr, dy.ptr, None))
    return dy.to_numpy(np.float32, (B, per))


def gating_expf(x: float) -> float:
    return L.lib().qnb_gating_expf(C.c_float(x))


__all__ = [n for n in dir() if not n.startswith("_")] + ["QnbError"]
