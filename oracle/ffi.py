"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes bindings of the two CPU oracles.

  Restatement  oracle/liboracle.so        plain-C restatement (qnet_oracle.c)
  Reference    oracle/_ref/libqnet_ref.so the unmodified reference + extern "C" shim

Both expose the same Python surface as paper_2209_15427_b200.ops (same argument
order, numpy arrays in the reference's NCHW layout) so a parity test can call
`oracle_impl.conv_forward(...)` and `ops.conv_forward(...)` on identical inputs.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "liboracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libqnet_ref.so")

FP32, FP16, INT8Q, INT16Q = 0, 1, 2, 3
NP_OF = {FP32: np.float32, FP16: np.uint16, INT8Q: np.uint8, INT16Q: np.uint16}


class QVals(C.Structure):
    _fields_ = [("f_min", C.c_double), ("f_max", C.c_double), ("scale", C.c_double),
                ("zero", C.c_int32), ("one", C.c_double), ("i_min", C.c_int64), ("i_max", C.c_int64)]

    def as_tuple(self):
        return (self.f_min, self.f_max, self.scale, self.zero, self.one, self.i_min, self.i_max)


class Requant(C.Structure):
    _fields_ = [("shift_bits", C.c_int32), ("mult", C.c_int64), ("shift", C.c_int32),
                ("in_zero", C.c_int64), ("out_zero", C.c_int64), ("out_min", C.c_int64),
                ("out_max", C.c_int64)]

    def as_tuple(self):
        return (self.shift_bits, self.mult, self.shift, self.in_zero, self.out_zero, self.out_min,
                self.out_max)


class ConvParams(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("out_channels", "kernel_h", "kernel_w", "stride_h",
                                         "stride_w", "pad_h", "pad_w", "groups", "bias_term")]


class OracleError(RuntimeError):
    pass


def build_restatement() -> None:
    """Compiles liboracle.so (gcc only; works on the GPU box too)."""
    if not os.path.exists(RESTATEMENT_SO) or os.path.getmtime(RESTATEMENT_SO) < os.path.getmtime(
            os.path.join(HERE, "qnet_oracle.c")):
        subprocess.run(["make", "-C", HERE, "restatement"], check=True, capture_output=True)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _qv(q):
    if q is None:
        return None
    if isinstance(q, QVals):
        return C.byref(q)
    if hasattr(q, "as_tuple"):
        return C.byref(QVals(*q.as_tuple()))
    return C.byref(QVals(*q))


def _conv_params(cp, has_bias):
    return ConvParams(cp["out_channels"], cp.get("kernel_h", 1), cp.get("kernel_w", 1), cp.get("stride_h", 1),
                      cp.get("stride_w", 1), cp.get("pad_h", 0), cp.get("pad_w", 0), cp.get("groups", 1),
                      1 if has_bias else 0)


class _Base:
    prefix = ""
    so_path = ""

    def __init__(self):
        if not os.path.exists(self.so_path):
            raise OracleError(f"{self.so_path} not built (make -C oracle)")
        self.lib = C.CDLL(self.so_path)
        p = self.prefix
        L = self.lib
        for name, res in (("round_half_even", C.c_double), ("requant_round", C.c_int64),
                          ("requant_clamp", C.c_int64), ("quantize_value", C.c_int64),
                          ("fp16_encode", C.c_uint16), ("fp16_decode", C.c_float),
                          ("gating_noise", C.c_float)):
            getattr(L, p + name).restype = res
        getattr(L, p + "round_half_even").argtypes = [C.c_double]
        getattr(L, p + "requant_round").argtypes = [C.c_int64, C.c_void_p]
        getattr(L, p + "requant_clamp").argtypes = [C.c_int64, C.c_void_p]
        getattr(L, p + "quantize_value").argtypes = [C.c_double, C.c_void_p]
        getattr(L, p + "fp16_encode").argtypes = [C.c_float]
        getattr(L, p + "fp16_decode").argtypes = [C.c_uint16]
        getattr(L, p + "gating_noise").argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int]

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _err(self):
        raise NotImplementedError

    def _check(self, st):
        if st != 0:
            raise OracleError(self._err())

    # ---- quantizer math
    def round_half_even(self, x):
        return self._fn("round_half_even")(float(x))

    def estimate_params(self, f_min, f_max, dtype):
        q = QVals()
        self._check(self._fn("estimate_params")(C.c_double(f_min), C.c_double(f_max), dtype, C.byref(q)))
        return q

    def estimate_from_observation(self, lo, hi, dtype):
        q = QVals()
        self._check(self._fn("estimate_from_observation")(C.c_double(lo), C.c_double(hi), dtype, C.byref(q)))
        return q

    def quantize_value(self, x, qv):
        return self._fn("quantize_value")(float(x), _qv(qv))

    def scale_quant_vals(self, *args):
        rq = Requant()
        if len(args) == 3:
            self._check(self._fn("scale_quant_vals2")(_qv(args[0]), _qv(args[1]), int(args[2]), C.byref(rq)))
        else:
            self._check(self._fn("scale_quant_vals3")(_qv(args[0]), _qv(args[1]), _qv(args[2]), int(args[3]),
                                                      C.byref(rq)))
        return rq

    def requant_round(self, acc, rq):
        return self._fn("requant_round")(int(acc), C.byref(Requant(*rq.as_tuple())))

    def requant_clamp(self, acc, rq):
        return self._fn("requant_clamp")(int(acc), C.byref(Requant(*rq.as_tuple())))

    def fp16_encode(self, x):
        return self._fn("fp16_encode")(C.c_float(x))

    def fp16_decode(self, h):
        return self._fn("fp16_decode")(int(h))

    def gating_noise(self, seed, sample, expert, stream):
        return self._fn("gating_noise")(seed, sample, expert, stream)

    # ---- tensor ops (same surface as paper_2209_15427_b200.ops)
    def quantize(self, x, qv, dtype):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(x.shape, NP_OF[dtype])
        r = self._fn("quantize")(_ptr(x), C.c_int64(x.size), _qv(qv), dtype, _ptr(out))
        if self.prefix == "ref_":
            self._check(r)
        return out

    def dequantize(self, q, dtype, qv):
        q = np.ascontiguousarray(q)
        out = np.empty(q.shape, np.float32)
        r = self._fn("dequantize")(_ptr(q), C.c_int64(q.size), dtype, _qv(qv), _ptr(out))
        if self.prefix == "ref_":
            self._check(r)
        return out

    def relu_quant(self, q, dtype, rq):
        q = np.ascontiguousarray(q)
        out = np.empty_like(q)
        r = self._fn("relu_quant")(_ptr(q), C.c_int64(q.size), dtype, C.byref(Requant(*rq.as_tuple())), _ptr(out))
        if self.prefix == "ref_":
            self._check(r)
        return out

    def relu_float(self, x, dtype, slope):
        x = np.ascontiguousarray(x)
        out = np.empty_like(x)
        r = self._fn("relu_float")(_ptr(x), C.c_int64(x.size), dtype, C.c_float(slope), _ptr(out))
        if self.prefix == "ref_":
            self._check(r)
        return out

    def cast_float(self, x, from_dtype, to_dtype):
        x = np.ascontiguousarray(x)
        out = np.empty(x.shape, NP_OF[to_dtype])
        r = self._fn("cast_float")(_ptr(x), C.c_int64(x.size), from_dtype, to_dtype, _ptr(out))
        if self.prefix == "ref_":
            self._check(r)
        return out

    def pool_max(self, x, dtype, kernel, stride):
        x = np.ascontiguousarray(x)
        N, Ch, H, W = x.shape
        oh, ow = (H - kernel) // stride + 1, (W - kernel) // stride + 1
        out = np.empty((N, Ch, max(oh, 0), max(ow, 0)), x.dtype)
        shape = (C.c_int64 * 4)(N, Ch, H, W)
        self._check(self._fn("pool_max")(_ptr(x), shape, dtype, C.c_int64(kernel), C.c_int64(stride), _ptr(out)))
        return out

    def softmax(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty_like(x)
        if self.prefix == "ref_":
            shape = (C.c_int64 * x.ndim)(*x.shape)
            self._check(self._fn("softmax")(_ptr(x), x.ndim, shape, _ptr(out)))
        else:
            N = x.shape[0]
            self._fn("softmax")(_ptr(x), C.c_int64(N), C.c_int64(x.size // N), _ptr(out))
        return out

    def lrn(self, x, local_size=5, alpha=1e-4, beta=0.75, k=1.0):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty_like(x)
        if self.prefix == "ref_":
            shape = (C.c_int64 * x.ndim)(*x.shape)
            self._check(self._fn("lrn")(_ptr(x), x.ndim, shape, C.c_int64(local_size), C.c_double(alpha),
                                        C.c_double(beta), C.c_double(k), _ptr(out)))
        else:
            N, Ch = x.shape[0], x.shape[1]
            self._fn("lrn")(_ptr(x), C.c_int64(N), C.c_int64(Ch), C.c_int64(x.size // (N * Ch)),
                            C.c_int64(local_size), C.c_double(alpha), C.c_double(beta), C.c_double(k), _ptr(out))
        return out

    def conv_forward(self, x, dtype, weight, w_dtype, bias, cp, in_qv=None, w_qv=None, out_qv=None,
                     shift_bits=0):
        x = np.ascontiguousarray(x)
        weight = np.ascontiguousarray(weight)
        b = np.ascontiguousarray(bias, dtype=np.float32) if bias is not None else None
        p = _conv_params(cp, b is not None)
        N, Ch, H, W = x.shape
        oh = (H + 2 * p.pad_h - p.kernel_h) // p.stride_h + 1
        ow = (W + 2 * p.pad_w - p.kernel_w) // p.stride_w + 1
        out = np.empty((N, p.out_channels, max(oh, 1), max(ow, 1)), NP_OF[dtype])
        os_ = (C.c_int64 * 4)()
        xs = (C.c_int64 * 4)(*x.shape)
        if self.prefix == "ref_":
            ws = (C.c_int64 * 4)(*weight.shape)
            self._check(self._fn("conv_forward")(_ptr(x), xs, dtype, _qv(in_qv), _ptr(weight), ws, w_dtype,
                                                 _qv(w_qv), _ptr(b), C.byref(p), _qv(out_qv), shift_bits,
                                                 _ptr(out), os_))
        else:
            self._check(self._fn("conv_forward")(_ptr(x), xs, dtype, _qv(in_qv), _ptr(weight), w_dtype, _qv(w_qv),
                                                 _ptr(b), C.byref(p), _qv(out_qv), shift_bits, _ptr(out), os_))
        return out

    def inner_product(self, x, dtype, weight, w_dtype, bias, out_features, in_qv=None, w_qv=None, out_qv=None,
                      shift_bits=0):
        x = np.ascontiguousarray(x)
        weight = np.ascontiguousarray(weight)
        b = np.ascontiguousarray(bias, dtype=np.float32) if bias is not None else None
        N = x.shape[0]
        K = x.size // max(N, 1)
        out = np.empty((N, out_features), NP_OF[dtype])
        if self.prefix == "ref_":
            shape = (C.c_int64 * x.ndim)(*x.shape)
            self._check(self._fn("inner_product")(_ptr(x), x.ndim, shape, dtype, _qv(in_qv), _ptr(weight),
                                                  w_dtype, _qv(w_qv), _ptr(b), C.c_int64(out_features),
                                                  _qv(out_qv), shift_bits, _ptr(out)))
        else:
            self._check(self._fn("inner_product")(_ptr(x), C.c_int64(N), C.c_int64(K), dtype, _qv(in_qv),
                                                  _ptr(weight), w_dtype, _qv(w_qv), _ptr(b),
                                                  C.c_int64(out_features), _qv(out_qv), shift_bits, _ptr(out)))
        return out

    def gating_select(self, x, wa, wb, wc, top_k, noise=False, seed=0, sample=0):
        x = np.ascontiguousarray(x, dtype=np.float32)
        wa, wb, wc = (np.ascontiguousarray(a, dtype=np.float32) for a in (wa, wb, wc))
        N, D = wa.shape
        q = np.empty(N, np.float32)
        p = np.empty(N, np.float32)
        idx = np.empty(top_k, np.int64)
        w = np.empty(top_k, np.float32)
        self._check(self._fn("gating_select")(_ptr(x), C.c_int64(D), _ptr(wa), _ptr(wb), _ptr(wc), C.c_int64(N),
                                              1 if noise else 0, C.c_uint64(seed), C.c_int64(sample),
                                              C.c_int64(top_k), _ptr(q), _ptr(p), _ptr(idx), _ptr(w)))
        return q, p, idx, w


class Restatement(_Base):
    """oracle/liboracle.so — the plain-C restatement."""

    prefix = "qo_"
    so_path = RESTATEMENT_SO

    def __init__(self):
        build_restatement()
        super().__init__()
        self.lib.qo_last_error.restype = C.c_char_p

    def _err(self):
        return self.lib.qo_last_error().decode()

    def requantize(self, q, in_dtype, rq, out_dtype):
        q = np.ascontiguousarray(q)
        out = np.empty(q.shape, NP_OF[out_dtype])
        self.lib.qo_requant_tensor(_ptr(q), C.c_int64(q.size), in_dtype, C.byref(Requant(*rq.as_tuple())),
                                   out_dtype, _ptr(out))
        return out

    def moe_combine(self, expert_out, idx, weights):
        E, B, per = expert_out.shape
        K = idx.shape[1]
        out = np.empty((B, per), np.float32)
        eo = np.ascontiguousarray(expert_out, dtype=np.float32)
        ii = np.ascontiguousarray(idx, dtype=np.int64)
        ww = np.ascontiguousarray(weights, dtype=np.float32)
        self.lib.qo_moe_combine(C.c_int64(B), C.c_int64(per), C.c_int64(K), _ptr(ii), _ptr(ww), _ptr(eo), _ptr(out))
        return out


class Reference(_Base):
    """oracle/_ref/libqnet_ref.so — the unmodified reference behind an extern C shim."""

    prefix = "ref_"
    so_path = REFERENCE_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_net_create.restype = C.c_void_p
        L.ref_net_create.argtypes = [C.c_char_p, C.c_int]
        L.ref_net_destroy.argtypes = [C.c_void_p]
        L.ref_net_graph_json.restype = C.c_char_p
        L.ref_net_graph_json.argtypes = [C.c_void_p]
        L.ref_override_precision_json.restype = C.c_char_p
        L.ref_override_precision_json.argtypes = [C.c_char_p, C.c_int]
        L.ref_validate_json.restype = C.c_char_p
        L.ref_validate_json.argtypes = [C.c_char_p]
        L.ref_plan_memory_peak.restype = C.c_int64
        L.ref_plan_memory_peak.argtypes = [C.c_char_p, C.c_int]
        L.ref_net_output_names.restype = C.c_char_p
        L.ref_net_output_names.argtypes = [C.c_void_p]
        L.ref_load_balance_loss.restype = C.c_double
        for fn in ("ref_net_set_param", "ref_net_param_info", "ref_net_param_data", "ref_net_set_range",
                   "ref_net_get_range", "ref_net_finalize", "ref_net_save", "ref_net_load", "ref_net_set_mode", "ref_net_blob_qvals",
                   "ref_net_forward", "ref_net_output_info", "ref_net_output_data", "ref_net_forward_mt"):
            getattr(L, fn).argtypes = None
        L.ref_net_set_range.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_double]

    def _err(self):
        return self.lib.ref_last_error().decode()

    def last_error(self):
        return self._err()

    def requantize(self, q, in_dtype, rq, out_dtype):
        out = np.empty(q.shape, NP_OF[out_dtype])
        flat_in = q.reshape(-1)
        flat = out.reshape(-1)
        for i in range(flat_in.size):
            flat[i] = self.requant_clamp(int(flat_in[i]) - rq.in_zero, rq)
        return out

    def load_balance_loss(self, counts, n_experts, top_k, batch):
        c = np.ascontiguousarray(counts, dtype=np.int64)
        return self.lib.ref_load_balance_loss(_ptr(c), C.c_int64(n_experts), C.c_int64(top_k), C.c_int64(batch))

    def moe_forward_fixed(self, inp, feats, wa, wb, wc, top_k, expert_out, mode=1, noise=False, seed=0):
        """moe_forward with the BatchFn seam bound to precomputed gating features and
        expert outputs (expert_out[e][s]); mode 0 = PER_SAMPLE, 1 = ALL_EXPERTS."""
        B = inp.shape[0]
        inp = np.ascontiguousarray(inp.reshape(B, -1), dtype=np.float32)
        E, _, per = expert_out.shape
        out = np.empty((B, per), np.float32)
        arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (feats, wa, wb, wc, expert_out)]
        self._check(self.lib.ref_moe_forward_fixed(
            C.c_int64(B), _ptr(inp), C.c_int64(inp.shape[1]), _ptr(arrs[0]), C.c_int64(arrs[1].shape[1]),
            _ptr(arrs[1]), _ptr(arrs[2]), _ptr(arrs[3]), C.c_int64(E), C.c_int64(top_k), 1 if noise else 0,
            C.c_uint64(seed), mode, _ptr(arrs[4]), C.c_int64(per), _ptr(out)))
        return out

    # ---- graph / Net
    def override_precision_json(self, text: str, dtype: int) -> str:
        r = self.lib.ref_override_precision_json(text.encode(), dtype)
        if r is None:
            raise OracleError(self._err())
        return r.decode()

    def validate_json(self, text: str):
        r = self.lib.ref_validate_json(text.encode())
        if r is None:
            raise OracleError(self._err())
        return [v for v in r.decode().split("\n") if v]

    def net(self, graph_json: str, precision: int = -1) -> "RefNet":
        return RefNet(self, graph_json, precision)


class RefNet:
    """A qnet::Net held by the reference shim (src/net.cpp)."""

    def __init__(self, ref: Reference, graph_json: str, precision: int = -1):
        self.ref = ref
        self.L = ref.lib
        self.h = self.L.ref_net_create(graph_json.encode(), precision)
        if not self.h:
            raise OracleError(ref._err())
        self.h = C.c_void_p(self.h)

    def __del__(self):
        try:
            if self.h:
                self.L.ref_net_destroy(self.h)
        except Exception:
            pass

    def graph_json(self) -> str:
        return self.L.ref_net_graph_json(self.h).decode()

    def set_param(self, name: str, arr: np.ndarray, dtype: int = FP32, qv=None):
        arr = np.ascontiguousarray(arr)
        shape = (C.c_int64 * max(arr.ndim, 1))(*arr.shape)
        self.ref._check(self.L.ref_net_set_param(self.h, name.encode(), dtype, arr.ndim, shape, _ptr(arr), _qv(qv)))

    def param(self, name: str):
        dt, nd, hq = C.c_int(), C.c_int(), C.c_int()
        shape = (C.c_int64 * 8)()
        qv = QVals()
        if not self.L.ref_net_param_info(self.h, name.encode(), C.byref(dt), C.byref(nd), shape, C.byref(qv),
                                         C.byref(hq)):
            return None, None
        arr = np.empty(tuple(shape[: nd.value]), NP_OF[dt.value])
        self.L.ref_net_param_data(self.h, name.encode(), _ptr(arr))
        return arr, (qv if hq.value else None)

    def set_range(self, key: str, lo: float, hi: float):
        self.ref._check(self.L.ref_net_set_range(self.h, key.encode(), lo, hi))

    def range(self, key: str):
        lo, hi = C.c_double(), C.c_double()
        if self.L.ref_net_get_range(self.h, key.encode(), C.byref(lo), C.byref(hi)):
            return lo.value, hi.value
        return None

    def finalize(self):
        self.ref._check(self.L.ref_net_finalize(self.h))

    def save(self, path: str):
        """save_model(net.to_model(), path) (src/model_store.cpp:123-175)."""
        self.ref._check(self.L.ref_net_save(self.h, path.encode()))

    def load(self, path: str):
        """net.load_weights(load_model(path)) (src/net.cpp:605-619)."""
        self.ref._check(self.L.ref_net_load(self.h, path.encode()))

    def set_mode(self, mode: int):
        """0 PASSIVE, 1 OBSERVE, 2 PSEUDO, 3 QUANTIZED."""
        self.ref._check(self.L.ref_net_set_mode(self.h, mode))

    def blob_qvals(self, blob: str):
        qv = QVals()
        return qv if self.L.ref_net_blob_qvals(self.h, blob.encode(), C.byref(qv)) else None

    def forward(self, input_name: str, x: np.ndarray, dtype: int = FP32):
        x = np.ascontiguousarray(x)
        shape = (C.c_int64 * x.ndim)(*x.shape)
        self.ref._check(self.L.ref_net_forward(self.h, input_name.encode(), dtype, x.ndim, shape, _ptr(x)))
        names = [n for n in self.L.ref_net_output_names(self.h).decode().split("\n") if n]
        outs = {}
        for n in names:
            dt, nd, hq = C.c_int(), C.c_int(), C.c_int()
            shp = (C.c_int64 * 8)()
            qv = QVals()
            self.L.ref_net_output_info(self.h, n.encode(), C.byref(dt), C.byref(nd), shp, C.byref(qv), C.byref(hq))
            arr = np.empty(tuple(shp[: nd.value]), NP_OF[dt.value])
            self.L.ref_net_output_data(self.h, n.encode(), _ptr(arr))
            outs[n] = (arr, dt.value, qv if hq.value else None)
        return outs


def forward_mt(nets, input_name: str, x: np.ndarray, output: str, out_per_bytes: int, dtype: int = FP32):
    """Batch forward split over len(nets) host threads, one reference Net each."""
    ref = nets[0].ref
    x = np.ascontiguousarray(x)
    shape = (C.c_int64 * x.ndim)(*x.shape)
    handles = (C.c_void_p * len(nets))(*[n.h.value for n in nets])
    out = np.empty(x.shape[0] * out_per_bytes, np.uint8)
    ref._check(ref.lib.ref_net_forward_mt(handles, len(nets), input_name.encode(), dtype, x.ndim, shape, _ptr(x),
                                          output.encode(), C.c_int64(out_per_bytes), _ptr(out)))
    return out


def have_reference() -> bool:
    return os.path.exists(REFERENCE_SO)
