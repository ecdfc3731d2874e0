"""ctypes binding of libqnb.so — the C-ABI declared in include/qnb.h.

The product path is this shared library and nothing else: if it is missing, or no
sm_100 device is present, every compute call raises.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# QNB_LIB_VARIANT=spin selects the A/B build with spinning mbarrier waits (profiling only)
LIB_PATH = os.path.join(_HERE, "libqnb_spin.so" if os.environ.get("QNB_LIB_VARIANT") == "spin" else "libqnb.so")

# qnet::DataType codes (include/qnet/datatypes.hpp:30-35)
FP32, FP16, INT8Q, INT16Q = 0, 1, 2, 3
DTYPE_NAMES = {FP32: "fp32", FP16: "fp16", INT8Q: "int8", INT16Q: "int16"}
DTYPE_BY_NAME = {"fp32": FP32, "float": FP32, "fp16": FP16, "half": FP16, "int8": INT8Q, "int16": INT16Q}

STATUS_NAMES = {
    0: "QNB_OK", 1: "QNB_E_ARG", 2: "QNB_E_SHAPE", 3: "QNB_E_GROUPS", 4: "QNB_E_EXTENT",
    5: "QNB_E_QVALS", 6: "QNB_E_DTYPE", 7: "QNB_E_RATIO", 8: "QNB_E_CUDA", 9: "QNB_E_OOM",
    10: "QNB_E_UNSUPPORTED", 11: "QNB_E_IO",
}


class QnbError(RuntimeError):
    """Raised for a non-OK qnb_status; .status holds the code, str() the reference message."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.status_name = STATUS_NAMES.get(status, str(status))


class QVals(C.Structure):
    """qnet::QuantizerValues (include/qnet/quantizer_values.hpp:32-42)."""

    _fields_ = [("f_min", C.c_double), ("f_max", C.c_double), ("scale", C.c_double),
                ("zero", C.c_int32), ("one", C.c_double), ("i_min", C.c_int64), ("i_max", C.c_int64)]

    def __repr__(self):
        return (f"QVals(f_min={self.f_min!r}, f_max={self.f_max!r}, scale={self.scale!r}, "
                f"zero={self.zero}, i_min={self.i_min}, i_max={self.i_max})")

    def as_tuple(self):
        return (self.f_min, self.f_max, self.scale, self.zero, self.one, self.i_min, self.i_max)


class Requant(C.Structure):
    """qnet::RequantParams (include/qnet/quantizer_values.hpp:59-67)."""

    _fields_ = [("shift_bits", C.c_int32), ("mult", C.c_int64), ("shift", C.c_int32),
                ("in_zero", C.c_int64), ("out_zero", C.c_int64), ("out_min", C.c_int64),
                ("out_max", C.c_int64)]

    def as_tuple(self):
        return (self.shift_bits, self.mult, self.shift, self.in_zero, self.out_zero, self.out_min,
                self.out_max)


class ConvParams(C.Structure):
    """qnet::ConvParams (include/qnet/ops.hpp:31-41)."""

    _fields_ = [(n, C.c_int64) for n in ("out_channels", "kernel_h", "kernel_w", "stride_h",
                                         "stride_w", "pad_h", "pad_w", "groups", "bias_term")]


class LayerDesc(C.Structure):
    """qnb_layer_desc (include/qnb.h)."""

    _fields_ = [
        ("kind", C.c_int32), ("mi_type", C.c_int32), ("d_type", C.c_int32), ("mo_type", C.c_int32),
        ("bottom", C.c_int32), ("top", C.c_int32), ("input_ndim", C.c_int32),
        ("input_shape", C.c_int64 * 4), ("conv", ConvParams),
        ("pool_kernel", C.c_int64), ("pool_stride", C.c_int64),
        ("lrn_local_size", C.c_int64), ("lrn_alpha", C.c_double), ("lrn_beta", C.c_double), ("lrn_k", C.c_double),
        ("negative_slope", C.c_float), ("num_output", C.c_int64), ("bias_term", C.c_int32),
        ("weight", C.c_void_p), ("weight_dtype", C.c_int32), ("weight_has_qv", C.c_int32),
        ("weight_qv", QVals), ("bias", C.c_void_p), ("top_has_qv", C.c_int32), ("top_qv", QVals),
        ("inspect_top", C.c_int32),
    ]


class Record(C.Structure):
    """qnb_record (include/qnb.h): one QCNM record."""

    _fields_ = [("name", C.c_char_p), ("dtype", C.c_int32), ("rank", C.c_int32), ("extents", C.c_int64 * 8),
                ("f_min", C.c_float), ("f_max", C.c_float), ("scale", C.c_float), ("zero", C.c_float),
                ("one", C.c_float), ("payload", C.c_void_p), ("payload_bytes", C.c_int64)]


class PlanOpts(C.Structure):
    _fields_ = [("max_batch", C.c_int64), ("use_cuda_graph", C.c_int32), ("flags", C.c_int32)]


class GraphDesc(C.Structure):
    """qnb_graph_desc (include/qnb.h)."""

    _fields_ = [("layers", C.POINTER(LayerDesc)), ("n_layers", C.c_int32), ("n_blobs", C.c_int32)]


class MoeOpts(C.Structure):
    """qnb_moe_opts (include/qnb.h)."""

    _fields_ = [("max_batch", C.c_int64), ("n_experts", C.c_int32), ("top_k", C.c_int32),
                ("noise_enabled", C.c_int32), ("seed", C.c_uint64), ("sample_offset", C.c_int64),
                ("in_dtype", C.c_int32), ("in_qv", QVals), ("top_dtype", C.c_int32), ("top_qv", QVals),
                ("in_per_sample", C.c_int64), ("out_per_sample", C.c_int64), ("gate_dim", C.c_int32),
                ("gate_a", C.c_void_p), ("gate_b", C.c_void_p), ("gate_c", C.c_void_p),
                ("use_cuda_graph", C.c_int32)]


_PLAN_SIGS = {
    "qnb_plan_create": (C.c_int, [C.POINTER(LayerDesc), C.c_int32, C.c_int32, C.POINTER(PlanOpts),
                                  C.POINTER(C.c_void_p)]),
    "qnb_plan_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32,
                                   C.c_void_p]),
    "qnb_plan_forward_dyn": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "qnb_plan_output_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int64)]),
    "qnb_plan_blob_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "qnb_plan_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64)]),
    "qnb_plan_observe": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.c_void_p]),
    "qnb_plan_destroy": (C.c_int, [C.c_void_p]),
    "qnb_moe_plan_create": (C.c_int, [C.POINTER(GraphDesc), C.POINTER(GraphDesc), C.POINTER(GraphDesc),
                                      C.POINTER(GraphDesc), C.POINTER(MoeOpts), C.POINTER(C.c_void_p)]),
    "qnb_moe_plan_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32,
                                       C.c_void_p]),
    "qnb_moe_plan_status": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]),
    "qnb_moe_plan_moe_output": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "qnb_moe_plan_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "qnb_moe_plan_destroy": (C.c_int, [C.c_void_p]),
    "qnb_group_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "qnb_group_create": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_uint8), C.c_int32, C.POINTER(C.c_void_p)]),
    "qnb_group_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
                                    C.c_void_p]),
    "qnb_group_allgather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "qnb_group_alltoallv": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_void_p]),
    "qnb_group_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "qnb_group_destroy": (C.c_int, [C.c_void_p]),
    "qnb_model_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "qnb_model_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "qnb_model_record": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(Record)]),
    "qnb_model_close": (C.c_int, [C.c_void_p]),
    "qnb_model_save": (C.c_int, [C.c_char_p, C.POINTER(Record), C.c_int64]),
    "qnb_plan_step_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "qnb_plan_profile": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p,
                                   C.POINTER(C.c_float)]),
}



_lib = None

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int
_D = C.c_double
_SIGS = {
    "qnb_abi_version": (_I32, []),
    "qnb_last_error": (C.c_char_p, []),
    "qnb_device_check": (_I32, [_I32]),
    "qnb_malloc": (_I32, [C.POINTER(_P), C.c_size_t]),
    "qnb_free": (_I32, [_P]),
    "qnb_memcpy_h2d": (_I32, [_P, _P, C.c_size_t, _P]),
    "qnb_memcpy_d2h": (_I32, [_P, _P, C.c_size_t, _P]),
    "qnb_stream_sync": (_I32, [_P]),
    "qnb_kernel_launch_count": (C.c_uint64, []),
    "qnb_round_half_even": (_D, [_D]),
    "qnb_estimate_params": (_I32, [_D, _D, _I32, C.POINTER(QVals)]),
    "qnb_estimate_from_observation": (_I32, [_D, _D, _I32, C.POINTER(QVals)]),
    "qnb_scale_quant_vals": (_I32, [C.POINTER(QVals), C.POINTER(QVals), _I32, C.POINTER(Requant)]),
    "qnb_scale_quant_vals3": (_I32, [C.POINTER(QVals), C.POINTER(QVals), C.POINTER(QVals), _I32,
                                     C.POINTER(Requant)]),
    "qnb_requant_clamp_host": (_I64, [_I64, C.POINTER(Requant)]),
    "qnb_quantize": (_I32, [_P, _I64, C.POINTER(QVals), _I32, _P, _P]),
    "qnb_dequantize": (_I32, [_P, _I64, _I32, C.POINTER(QVals), _P, _P]),
    "qnb_requantize": (_I32, [_P, _I64, _I32, C.POINTER(Requant), _I32, _P, _P]),
    "qnb_relu_quant": (_I32, [_P, _I64, _I32, C.POINTER(Requant), _P, _P]),
    "qnb_relu_float": (_I32, [_P, _I64, _I32, C.c_float, _P, _P]),
    "qnb_cast_float": (_I32, [_P, _I64, _I32, _I32, _P, _P]),
    "qnb_pool_max": (_I32, [_P, C.POINTER(_I64), _I32, _I64, _I64, _P, _P]),
    "qnb_lrn": (_I32, [_P, _I64, _I64, _I64, _I64, _D, _D, _D, _P, _P]),
    "qnb_softmax": (_I32, [_P, _I64, _I64, _P, _P]),
    "qnb_conv_forward": (_I32, [_P, C.POINTER(_I64), _I32, C.POINTER(QVals), _P, _I32,
                                C.POINTER(QVals), _P, C.POINTER(ConvParams), C.POINTER(QVals), _I32,
                                _P, C.POINTER(_I64), _P]),
    "qnb_inner_product": (_I32, [_P, _I64, _I64, _I32, C.POINTER(QVals), _P, _I32, C.POINTER(QVals),
                                 _P, _I64, C.POINTER(QVals), _I32, _P, _P]),
    "qnb_moe_gate": (_I32, [_P, _I64, _I64, _P, _P, _P, _I64, _I64, _I32, C.c_uint64, _P, _P, _P]),
    "qnb_gating_expf": (C.c_float, [C.c_float]),
    "qnb_moe_gate_at": (_I32, [_P, _I64, _I64, _P, _P, _P, _I64, _I64, _I32, C.c_uint64, _I64, _P, _P, _P]),
    "qnb_gating_noise": (C.c_float, [C.c_uint64, _I64, _I64, _I32]),
    "qnb_moe_combine": (_I32, [_P, _I64, _I64, _I64, _P, _P, _P, _P]),
    "qnb_moe_route": (_I32, [_P, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
    "qnb_gather_rows": (_I32, [_P, _I64, _P, _I64, _P, _P]),
    "qnb_moe_combine_rows": (_I32, [_P, _I64, _P, _P, _I64, _I64, _I32, C.POINTER(QVals), _P, _P]),
}
_SIGS.update(_PLAN_SIGS)


def lib() -> C.CDLL:
    """Loads libqnb.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise QnbError(8, f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the B200 backend has no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().qnb_last_error().decode(errors="replace")
        raise QnbError(status, msg)


def exported_symbols():
    return list(_SIGS)
