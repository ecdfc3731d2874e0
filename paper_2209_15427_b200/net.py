"""Host-side mirror of qnet::Net (include/qnet/net.hpp:44-92) whose forward runs the
compiled B200 plan (qnb_plan_* in include/qnb.h).

    net = Net(override_precision(alexnet(), "int8"))
    for name, arr in params.items(): net.set_param(name, arr)
    for key, (lo, hi) in ranges.items(): net.set_range(key, lo, hi)
    net.finalize_quantizers()                  # src/net.cpp:211-248
    net.set_quant_mode(QUANTIZED)              # src/net.cpp:250-275
    out = net.forward({"data": images})        # src/net.cpp:305-330 -> {"prob": ...}

Parameters, calibration ranges, finalization and the error messages follow the
reference.  Weight quantization during finalize runs on the GPU (qnb_quantize).
"""
from __future__ import annotations

import copy
import ctypes as C

import numpy as np

from . import _lib as L
from . import graph as G
from . import ops
from ._lib import QnbError, QVals, check

PASSIVE, OBSERVE, PSEUDO, QUANTIZED = 0, 1, 2, 3


from ._lib import LayerDesc, PlanOpts  # noqa: E402


def _plan_lib():
    return L.lib()


NP_OF = {0: np.float32, 1: np.uint16, 2: np.uint8, 3: np.uint16}


class Plan:
    """A compiled device plan (qnb_plan) for one calibrated chain graph."""

    OBSERVE = 1      # QNB_PLAN_OBSERVE: every top materialised (no fusion)
    EXACT_FLOAT = 2  # QNB_PLAN_EXACT_FLOAT: FP32 conv / IP in the reference's exact arithmetic

    def __init__(self, descs, n_blobs, keep_alive, max_batch, use_cuda_graph=True, blob_ids=None, flags=0):
        self._keep = keep_alive
        self.max_batch = max_batch
        self.blob_ids = blob_ids or {}
        self.n_blobs = n_blobs
        arr = (LayerDesc * len(descs))(*descs)
        opts = PlanOpts(max_batch, 1 if use_cuda_graph else 0, flags)
        self.h = C.c_void_p()
        lib = _plan_lib()
        check(lib.qnb_plan_create(arr, len(descs), n_blobs, C.byref(opts), C.byref(self.h)))
        dt, nd = C.c_int32(), C.c_int32()
        shape = (C.c_int64 * 4)()
        check(lib.qnb_plan_output_info(self.h, C.byref(dt), C.byref(nd), shape))
        self.out_dtype, self.out_ndim = dt.value, nd.value
        self.out_shape = tuple(shape[: nd.value])
        self._keep = None  # host parameter copies are no longer needed

    def stats(self):
        k, a, w = C.c_int64(), C.c_int64(), C.c_int64()
        check(_plan_lib().qnb_plan_stats(self.h, C.byref(k), C.byref(a), C.byref(w)))
        return {"kernels_per_forward": k.value, "arena_bytes": a.value, "weight_bytes": w.value}

    STEP_KINDS = {0: "pack_input", 1: "igemm", 2: "pool", 3: "pool_lrn", 4: "convert", 5: "softmax", 7: "conv_pool",
                  6: "unpack"}

    def steps(self):
        """[(layer index, kind name, ops, bytes)] per step at max_batch."""
        n = self.stats()["kernels_per_forward"]
        out = []
        for i in range(n):
            lay, kind, ops_, by = C.c_int32(), C.c_int32(), C.c_double(), C.c_double()
            check(_plan_lib().qnb_plan_step_info(self.h, i, C.byref(lay), C.byref(kind), C.byref(ops_),
                                                 C.byref(by)))
            out.append((lay.value, self.STEP_KINDS.get(kind.value, "?"), ops_.value, by.value))
        return out

    def profile(self, in_ptr: int, out_ptr: int, batch: int, reps: int = 3, stream: int = 0):
        """Mean ms per step (eager launches, CUDA events between steps)."""
        n = self.stats()["kernels_per_forward"]
        ms = (C.c_float * n)()
        check(_plan_lib().qnb_plan_profile(self.h, C.c_void_p(in_ptr), batch, C.c_void_p(out_ptr), reps,
                                           C.c_void_p(stream), ms))
        return list(ms)

    def forward_host(self, x: np.ndarray) -> np.ndarray:
        """Host buffers in and out (copies inside the call)."""
        x = np.ascontiguousarray(x)
        b = x.shape[0]
        out = np.empty((b,) + self.out_shape[1:], NP_OF[self.out_dtype])
        check(_plan_lib().qnb_plan_forward(self.h, x.ctypes.data_as(C.c_void_p), b, 1,
                                           out.ctypes.data_as(C.c_void_p), 1, None))
        check(L.lib().qnb_stream_sync(None))
        return out

    def forward_device(self, in_ptr: int, out_ptr: int, batch: int, stream: int = 0,
                       in_host: bool = False, out_host: bool = False) -> None:
        """Raw pointers (device by default), stream-ordered, no synchronisation."""
        check(_plan_lib().qnb_plan_forward(self.h, C.c_void_p(in_ptr), batch, 1 if in_host else 0,
                                           C.c_void_p(out_ptr), 1 if out_host else 0, C.c_void_p(stream)))

    def forward_dyn(self, in_ptr: int, out_ptr: int, batch_cap: int, dyn_ptr: int, stream: int = 0) -> None:
        """qnb_plan_forward_dyn: launched at batch_cap, processes *dyn_ptr (int32, device) images."""
        check(_plan_lib().qnb_plan_forward_dyn(self.h, C.c_void_p(in_ptr), batch_cap, C.c_void_p(dyn_ptr),
                                               C.c_void_p(out_ptr), C.c_void_p(stream)))

    def observe_host(self, x: np.ndarray):
        """qnb_plan_observe on a host batch: (output, {blob id: (min, max)})."""
        x = np.ascontiguousarray(x)
        b = x.shape[0]
        lib = L.lib()
        d = C.c_void_p()
        check(lib.qnb_malloc(C.byref(d), x.nbytes))
        try:
            check(lib.qnb_memcpy_h2d(d, x.ctypes.data_as(C.c_void_p), x.nbytes, None))
            lo = (C.c_double * self.n_blobs)()
            hi = (C.c_double * self.n_blobs)()
            check(_plan_lib().qnb_plan_observe(self.h, d, b, lo, hi, None))
            out = self.forward_host(x)
        finally:
            lib.qnb_free(d)
        seen = {i: (lo[i], hi[i]) for i in range(self.n_blobs) if lo[i] == lo[i]}
        return out, seen

    def blob(self, name: str, shape=None):
        """Reads a materialised blob's interior back (NHWC -> reference NCHW)."""
        ptr = C.c_void_p()
        lay = (C.c_int64 * 8)()
        check(_plan_lib().qnb_plan_blob_info(self.h, self.blob_ids[name], C.byref(ptr), lay))
        if not ptr.value:
            return None
        n, h, w, cp, hh, hw, wx, es = list(lay)
        raw = np.empty(n * (h + 2 * hh) * (w + 2 * hw + wx) * cp * es, np.uint8)
        check(L.lib().qnb_memcpy_d2h(raw.ctypes.data_as(C.c_void_p), ptr, raw.nbytes, None))
        check(L.lib().qnb_stream_sync(None))
        return raw, (n, h, w, cp, hh, hw, wx, es)

    def __del__(self):
        try:
            if self.h:
                _plan_lib().qnb_plan_destroy(self.h)
        except Exception:
            pass


class Net:
    """qnet::Net surface backed by the B200 plan."""

    def __init__(self, graph: dict):
        self.graph = G.normalized(graph)
        self.blobs = G.infer_blobs(self.graph)
        self.aliases = G.range_aliases(self.graph)
        if any(l["kind"] == "moe" for l in self.graph["layers"]):
            raise QnbError(10, "MOE graphs run through paper_2209_15427_b200.moe.MoeNet")
        self.params = {}       # name -> (array, dtype code, qv or None)
        self.ranges = {}       # range key -> (lo, hi)
        self.blob_qv = {}
        self.mode = PASSIVE
        self._plans = {}

    # ---- parameters / ranges (src/net.cpp:140-209)
    def set_param(self, name, arr, dtype=0, qv=None):
        self.params[name] = (np.ascontiguousarray(arr), dtype, qv)
        self._plans.clear()

    def param(self, name):
        return self.params.get(name)

    def set_range(self, key, lo, hi):
        self.ranges[G.range_key(self.aliases, key)] = (float(lo), float(hi))
        self._plans.clear()

    def range(self, key):
        return self.ranges.get(G.range_key(self.aliases, key))

    def finalize_quantizers(self):
        """src/net.cpp:211-248."""
        for l in self.graph["layers"]:
            if l["kind"] not in ("conv", "inner_product") or l["compute_data_type"] not in G.QUANT:
                continue
            dt = G.DTYPE_CODE[l["compute_data_type"]]
            wkey = l["name"] + ".weight"
            if wkey not in self.params or self.params[wkey][1] != 0:
                continue
            w = self.params[wkey][0]
            if wkey in self.ranges:
                lo, hi = self.ranges[wkey]
            else:
                lo, hi = float(w.min()), float(w.max())
            qv = ops.estimate_from_observation(lo, hi, dt)
            self.params[wkey] = (ops.quantize(w, qv, dt), dt, qv)
        for b, info in self.blobs.items():
            if info["dtype"] not in G.QUANT:
                continue
            r = self.ranges.get(G.range_key(self.aliases, b))
            if r is not None:
                self.blob_qv[b] = ops.estimate_from_observation(r[0], r[1], G.DTYPE_CODE[info["dtype"]])
        self._plans.clear()

    def set_quant_mode(self, mode):
        """src/net.cpp:250-275 (OBSERVE and PSEUDO are host-calibration modes, not the B200 path)."""
        if mode in (QUANTIZED, PSEUDO):
            for b, info in self.blobs.items():
                if info["dtype"] in G.QUANT and b not in self.blob_qv:
                    raise QnbError(5, "quantizer not finalized: " + G.range_key(self.aliases, b))
            for l in self.graph["layers"]:
                if l["kind"] in ("conv", "inner_product") and l["compute_data_type"] in G.QUANT:
                    p = self.params.get(l["name"] + ".weight")
                    if p is not None and p[1] != G.DTYPE_CODE[l["compute_data_type"]]:
                        raise QnbError(5, "quantizer not finalized: " + l["name"] + ".weight")
        self.mode = mode

    # ---- model store (src/net.cpp:546-619)
    def to_model(self):
        """Net::to_model: parameter records in layer order (FP16 layers' FP32 weights
        narrowed), then one "blob:<key>" record per recorded range, keys sorted."""
        from .model_store import Model, ParamRecord, set_record_qvals
        recs = []
        for l in self.graph["layers"]:
            if l["kind"] not in ("conv", "inner_product"):
                continue
            bias = (l["conv"].get("bias_term", True) if l["kind"] == "conv" else l.get("bias_term", True))
            for name in [l["name"] + ".weight"] + ([l["name"] + ".bias"] if bias else []):
                p = self.params.get(name)
                if p is None:
                    continue
                arr, dt, qv = p
                is_weight = name.endswith(".weight")
                if is_weight and l["compute_data_type"] in G.QUANT and dt != G.DTYPE_CODE[l["compute_data_type"]]:
                    raise QnbError(5, "quantizer not finalized: " + name)
                if is_weight and l["compute_data_type"] == G.FP16 and dt == 0:
                    arr, dt = ops.cast_float(np.ascontiguousarray(arr, np.float32), 0, 1), 1
                arr = np.ascontiguousarray(arr, NP_OF[dt])
                r = ParamRecord(name, dt, tuple(arr.shape), payload=arr.view(np.uint8).reshape(-1))
                if qv is not None:
                    set_record_qvals(r, qv)
                recs.append(r)
        for key in sorted(self.ranges):
            lo, hi = self.ranges[key]
            recs.append(ParamRecord("blob:" + key, 0, (0,), float(np.float32(lo)), float(np.float32(hi))))
        return Model(recs)

    def load_weights(self, model) -> None:
        """Net::load_weights: "blob:" records set ranges, the others set parameters (with
        their quantizer values when the record is calibrated).  Parameter arrays are views
        into the model's file mapping."""
        from .model_store import record_qvals
        for r in model.records:
            if r.name.startswith("blob:"):
                self.set_range(r.name[5:], r.f_min, r.f_max)
                continue
            self.set_param(r.name, r.array(), r.dtype, record_qvals(r) if r.scale > 0 else None)
        self._model_keepalive = model

    def blob_qvals(self, blob):
        return self.blob_qv.get(blob)

    # ---- compilation
    def layer_descs(self):
        ids = {}
        for l in self.graph["layers"]:
            for b in l.get("bottom", []) + l["top"]:
                ids.setdefault(b, len(ids))
        descs, keep = [], []
        for l in self.graph["layers"]:
            d = LayerDesc()
            d.kind = G.KIND_CODE[l["kind"]]
            d.mi_type = G.DTYPE_CODE[l["bottom_data_type"]]
            d.d_type = G.DTYPE_CODE[l["compute_data_type"]]
            d.mo_type = G.DTYPE_CODE[l["top_data_type"]]
            d.bottom = ids[l["bottom"][0]] if l.get("bottom") else -1
            d.top = ids[l["top"][0]]
            k = l["kind"]
            if k == "input":
                d.input_ndim = len(l["input_shape"])
                for i, v in enumerate(l["input_shape"]):
                    d.input_shape[i] = v
            if k == "conv":
                c = l["conv"]
                d.conv = L.ConvParams(c["out_channels"], c.get("kernel_h", 1), c.get("kernel_w", 1),
                                      c.get("stride_h", 1), c.get("stride_w", 1), c.get("pad_h", 0),
                                      c.get("pad_w", 0), c.get("groups", 1), 1 if c.get("bias_term", True) else 0)
                d.bias_term = d.conv.bias_term
            if k == "pool":
                d.pool_kernel, d.pool_stride = l["pool"]["kernel"], l["pool"]["stride"]
            if k == "lrn":
                p = l.get("lrn", {})
                d.lrn_local_size = p.get("local_size", 5)
                d.lrn_alpha, d.lrn_beta, d.lrn_k = p.get("alpha", 1e-4), p.get("beta", 0.75), p.get("k", 1.0)
            if k == "relu":
                d.negative_slope = l.get("negative_slope", 0.0)
            if k == "inner_product":
                d.num_output = l["num_output"]
                d.bias_term = 1 if l.get("bias_term", True) else 0
            if k in ("conv", "inner_product"):
                w = self.params.get(l["name"] + ".weight")
                if w is None:
                    raise QnbError(1, "missing parameter: " + l["name"] + ".weight")
                arr, dt, qv = w
                if dt == 0 and l["compute_data_type"] == G.FP16:
                    pass  # fp32 weights feed the f16 MMA after rounding in the packer
                keep.append(arr)
                d.weight = arr.ctypes.data
                d.weight_dtype = dt
                if qv is not None:
                    d.weight_has_qv = 1
                    d.weight_qv = QVals(*qv.as_tuple()) if hasattr(qv, "as_tuple") else qv
                if d.bias_term:
                    b = self.params.get(l["name"] + ".bias")
                    if b is None:
                        raise QnbError(1, "missing parameter: " + l["name"] + ".bias")
                    barr = np.ascontiguousarray(b[0], dtype=np.float32)
                    keep.append(barr)
                    d.bias = barr.ctypes.data
            top = l["top"][0]
            d.inspect_top = 1 if top in self.graph.get("inspect", ()) else 0
            if l.get("pseudo_qv") is not None:
                d.top_has_qv = 1
                d.top_qv = QVals(*l["pseudo_qv"].as_tuple())
            if l["top_data_type"] in G.QUANT:
                qv = self.blob_qv.get(top)
                if qv is None:
                    raise QnbError(5, "quantizer not finalized: " + G.range_key(self.aliases, top))
                d.top_has_qv = 1
                d.top_qv = QVals(*qv.as_tuple())
            descs.append(d)
        return descs, len(ids), keep, ids

    def compile(self, max_batch: int, use_cuda_graph: bool = True) -> Plan:
        descs, n_blobs, keep, ids = self.layer_descs()
        return Plan(descs, n_blobs, keep, max_batch, use_cuda_graph, ids)

    def plan(self, batch: int) -> Plan:
        if batch not in self._plans:
            self._plans[batch] = self.compile(batch)
        return self._plans[batch]

    def observe_graph(self) -> dict:
        """The float execution Net::forward runs in OBSERVE mode (src/net.cpp:332-376): every
        layer in FP32, QUANTIZER / DROPOUT layers numeric no-ops.  QUANTIZER layers are dropped
        and their consumers rewired to the quantizer's bottom; the dropped tops share their
        bottom's range key (graph range_aliases), so the recorded ranges are the same."""
        g = copy.deepcopy(self.graph)
        ren, layers = {}, []
        for l in g["layers"]:
            if l.get("bottom"):
                l["bottom"] = [ren.get(b, b) for b in l["bottom"]]
            if l["kind"] == "quantizer":
                ren[l["top"][0]] = l["bottom"][0]
                continue
            l["bottom_data_type"] = l["compute_data_type"] = l["top_data_type"] = G.FP32
            layers.append(l)
        g["layers"] = layers
        return g

    def pseudo_graph(self) -> dict:
        """The execution Net::forward runs in PSEUDO mode (src/net.cpp:305-330, 379-389):
        the float execution of observe_graph() with every top fake-quantized onto its
        declared type (pseudo_quantize, src/quantizer.cpp:141-153; FP16 tops round through
        half).  Each fake-quant is a QUANTIZER layer with FP32 bottom/top and the declared
        type as compute type, carrying the blob's grid; a dropped QUANTIZER's fake-quant
        lands on its bottom's value, which only it consumes (chain graphs)."""
        g = copy.deepcopy(self.graph)
        ren, layers = {}, []

        def fake(blob, cur):
            dt = self.blobs[blob]["dtype"]
            if dt == G.FP32:
                return cur
            qv = None
            if dt in G.QUANT:
                qv = self.blob_qv.get(blob)
                if qv is None:
                    raise QnbError(5, "quantizer not finalized: " + G.range_key(self.aliases, blob))
            top = blob + "__pseudo"
            layers.append({"name": top, "kind": "quantizer", "bottom": [cur], "top": [top],
                           "bottom_data_type": G.FP32, "compute_data_type": dt, "top_data_type": G.FP32,
                           "pseudo_qv": qv})
            return top

        for l in g["layers"]:
            if l.get("bottom"):
                l["bottom"] = [ren.get(b, b) for b in l["bottom"]]
            top = l["top"][0]
            if l["kind"] == "quantizer":
                ren[top] = fake(top, l["bottom"][0])
                continue
            l["bottom_data_type"] = l["compute_data_type"] = l["top_data_type"] = G.FP32
            layers.append(l)
            ren[top] = fake(top, top)
        g["layers"] = layers
        sink = G.sinks(self.graph)[-1]
        return g, ren.get(sink, sink)

    def _float_plan(self, graph: dict, batch: int, flags: int = 0) -> Plan:
        """A plan over an all-FP32 execution graph with param_float() weights
        (src/net.cpp:183-196: finalized weights dequantize)."""
        saved, stash = self.graph, {}
        self.graph = graph
        try:
            for l in graph["layers"]:
                if l["kind"] in ("conv", "inner_product"):
                    w = self.params.get(l["name"] + ".weight")
                    if w is not None and w[1] != 0:
                        stash[l["name"] + ".weight"] = w
                        self.params[l["name"] + ".weight"] = (ops.dequantize(w[0], w[1], w[2]), 0, None)
            descs, n_blobs, keep, ids = self.layer_descs()
        finally:
            self.params.update(stash)
            self.graph = saved
        return Plan(descs, n_blobs, keep, batch, False, ids, flags=flags)

    def observe(self, x: np.ndarray) -> np.ndarray:
        """Net::forward in OBSERVE mode on the device: FP32 execution (exact reference arithmetic) and a
        min / max reduction per blob (observe(), src/quantizer.cpp:58-68); the ranges widen the
        ones already recorded (src/net.cpp:206-209)."""
        if x.dtype.kind not in "f":
            raise QnbError(10, "OBSERVE on the device takes float inputs")
        x = x.astype(np.float32)
        plan = self._float_plan(self.observe_graph(), x.shape[0], Plan.OBSERVE | Plan.EXACT_FLOAT)
        out, seen = plan.observe_host(x)
        for name, i in plan.blob_ids.items():
            if i not in seen:
                continue
            lo, hi = seen[i]
            key = G.range_key(self.aliases, name)
            if key in self.ranges:
                plo, phi = self.ranges[key]
                lo, hi = min(lo, plo), max(hi, phi)
            self.ranges[key] = (float(lo), float(hi))
        self._plans.clear()
        return out

    def pseudo(self, x: np.ndarray) -> np.ndarray:
        """Net::forward in PSEUDO mode on the device (fake-quant accuracy studies)."""
        if x.dtype.kind not in "f":
            raise QnbError(10, "PSEUDO on the device takes float inputs")
        x = x.astype(np.float32)
        key = ("pseudo", x.shape[0])
        if key not in self._plans:
            g, _ = self.pseudo_graph()
            self._plans[key] = self._float_plan(g, x.shape[0], Plan.EXACT_FLOAT)
        return self._plans[key].forward_host(x)

    @staticmethod
    def _input_dtype(x: np.ndarray, inl: dict) -> np.ndarray:
        """The INPUT layer of run_layer_typed (src/net.cpp:394-405): the plan reads the
        layer's mo_type; float inputs are cast to it, anything else must already be it."""
        want = G.DTYPE_CODE[inl["top_data_type"]]
        if want == 0 and x.dtype.kind == "f":
            return np.ascontiguousarray(x, np.float32)
        if want == 1 and x.dtype.kind == "f":  # FP16 tensors travel as raw uint16 bits
            return np.ascontiguousarray(x, np.float16).view(np.uint16)
        if x.dtype == NP_OF[want]:
            return x
        raise QnbError(6, "dtype mismatch at blob " + inl["top"][0])

    def forward(self, inputs: dict) -> dict:
        """src/net.cpp:305-330: returns {sink: tensor} in the reference layout."""
        name = G.input_name(self.graph)
        if name not in inputs:
            raise QnbError(1, "missing input: " + name)
        x = np.ascontiguousarray(inputs[name])
        inl = next(l for l in self.graph["layers"] if l["kind"] == "input")
        want = inl["input_shape"]
        if x.ndim != len(want) or list(x.shape[1:]) != list(want[1:]):
            raise QnbError(2, "shape mismatch")
        x = self._input_dtype(x, inl)
        if self.mode == OBSERVE:
            return {G.sinks(self.graph)[-1]: self.observe(x)}
        if self.mode == PSEUDO:
            return {G.sinks(self.graph)[-1]: self.pseudo(x)}
        out = self.plan(x.shape[0]).forward_host(x)
        return {G.sinks(self.graph)[-1]: out}
