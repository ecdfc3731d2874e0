"""Mixture-of-experts network on the B200: the host mirror of qnet::Net for graphs with
a MOE layer (Net::run_moe src/net.cpp:510-544 + moe_forward src/moe.cpp:165-252).

    net = MoeNet(override_precision(alexnet_moe(), "int8"))
    net.set_param("moe.expert3.e_conv1.weight", w) ...      # dotted names, net.hpp:36-40
    net.set_range("moe.gating.g_conv", lo, hi) ...
    net.finalize_quantizers(); net.set_quant_mode(QUANTIZED)
    out = net.forward({"data": images})                      # {"prob": ...}

Device pipeline of one forward (every arrow is a libqnb.so call on one stream):

    trunk plan -> int8 T (the MoE bottom blob, NCHW)
    qnb_dequantize(T) -> F                     run_layer_typed MOE: dequantize(*in)
    gating plan(F) -> feats (FP32, B x D)      gating_fn
    qnb_moe_gate -> idx, w (B x K)             gating_logits / gating_probs / select_topk
    qnb_moe_route -> pairs grouped per expert  PER_SAMPLE dispatch (== ALL_EXPERTS, moe.hpp:28-33)
    qnb_gather_rows(T) -> S (int8 pair rows)
      [N ranks: all-to-all of S to the experts' owners; the parent grid is identical on
       every rank, so the receiver's dequantize is bit-identical]
    qnb_dequantize(S) -> X; expert plan e on its contiguous rows -> Y
      [N ranks: all-to-all of Y back]
    qnb_moe_combine_rows(Y) -> M               mixing in selection order + quantize to the MoE top grid
    tail plan(M) -> sink

Expert plans run eagerly (their batch is data dependent); trunk, gating and tail plans
replay CUDA graphs.
"""
from __future__ import annotations

import ctypes as C
import re

import numpy as np

from . import _lib as L
from . import graph as G
from ._lib import QnbError, QVals, check
from .net import NP_OF, QUANTIZED, Net

_NESTED = re.compile(r"^([^.]+)\.(gating|expert(\d+))\.(.+)$")


def split_moe_graph(graph: dict):
    """(trunk, moe_layer, tail) chain graphs around the single MOE layer.  The tail
    starts with an INPUT layer whose top is the MoE top blob (same name, dtype)."""
    g = G.normalized(graph)
    layers = g["layers"]
    idx = [i for i, l in enumerate(layers) if l["kind"] == "moe"]
    if len(idx) != 1:
        raise QnbError(10, "MoeNet supports graphs with exactly one MOE layer")
    i = idx[0]
    moe = layers[i]
    blobs = G.infer_blobs(g)
    top = moe["top"][0]
    al = dict(g.get("range_aliases", {}))
    trunk = {"name": g.get("name", "") + "_trunk", "layers": layers[:i], "range_aliases": al}
    tin = {"name": top, "kind": "input", "top": [top], "input_shape": [1] + list(blobs[top]["shape"][1:]),
           "bottom_data_type": moe["top_data_type"], "compute_data_type": moe["top_data_type"],
           "top_data_type": moe["top_data_type"]}
    tail = {"name": g.get("name", "") + "_tail", "layers": [tin] + layers[i + 1:], "range_aliases": al}
    return trunk, moe, tail


class ExpertExchange:
    """Expert-parallel all-to-all of routed (sample, expert) pairs.

    Experts are placed contiguously, n_experts / world_size per rank.  `dispatch`
    takes this rank's pair rows grouped by global expert (qnb_moe_route order) and the
    per-expert counts, and returns the rows this rank's experts must process, grouped
    by local expert, plus per-local-expert counts.  `combine` returns the expert
    outputs to their home ranks in the original pair order.  Works with any
    torch.distributed backend (NCCL on the B200s, gloo in the CPU tests); `gather` is
    the row-permutation primitive (qnb_gather_rows on the device)."""

    def __init__(self, n_experts: int, rank: int, world: int, gather=None):
        if n_experts % world:
            raise QnbError(1, "n_experts must be divisible by the number of ranks")
        self.E, self.rank, self.world = n_experts, rank, world
        self.per_rank = n_experts // world
        self.gather = gather or (lambda t, rows: t.index_select(0, rows))

    def owner(self, e: int) -> int:
        return e // self.per_rank

    @staticmethod
    def plan(counts_all: np.ndarray, rank: int, per_rank: int):
        """Host bookkeeping from the (world x E) count matrix (row r = rank r's counts).
        Returns send splits, recv splits, and the permutation regrouping the received
        rows (ordered source-major) by local expert."""
        world, E = counts_all.shape
        send = [int(counts_all[rank, r * per_rank:(r + 1) * per_rank].sum()) for r in range(world)]
        local = counts_all[:, rank * per_rank:(rank + 1) * per_rank]  # (world, per_rank)
        recv = [int(local[s].sum()) for s in range(world)]
        src_off = np.concatenate([[0], np.cumsum(recv)[:-1]]).astype(np.int64)
        perm = []
        for e in range(per_rank):
            for s in range(world):
                start = src_off[s] + int(local[s, :e].sum())
                perm.extend(range(start, start + int(local[s, e])))
        local_counts = local.sum(axis=0).astype(np.int64)
        return send, recv, np.asarray(perm, np.int64), local_counts

    def dispatch(self, rows, counts: np.ndarray):
        import torch
        import torch.distributed as dist
        dev = rows.device
        c = torch.as_tensor(np.asarray(counts, np.int64), device=dev)
        allc = [torch.empty_like(c) for _ in range(self.world)]
        dist.all_gather(allc, c)
        counts_all = np.stack([t.cpu().numpy() for t in allc])
        send, recv, perm, local_counts = self.plan(counts_all, self.rank, self.per_rank)
        out = rows.new_empty((sum(recv),) + tuple(rows.shape[1:]))
        dist.all_to_all_single(out, rows.contiguous(), recv, send)
        self._state = (send, recv, perm)
        p = torch.as_tensor(perm, device=dev)
        grouped = self.gather(out, p) if len(perm) else out
        return grouped, local_counts

    def run(self, rows, counts: np.ndarray, expert_fn):
        """The expert-parallel step of one MoE forward: dispatch this rank's routed rows
        (grouped by global expert, `counts` per expert) to the experts' owners, run
        `expert_fn(e, rows_e) -> outputs` on the rows each local expert received, and return
        the outputs to their home ranks in the original pair order."""
        grouped, local_counts = self.dispatch(rows, counts)
        outs, off = [], 0
        for j in range(self.per_rank):
            c = int(local_counts[j])
            e = self.rank * self.per_rank + j
            outs.append(expert_fn(e, grouped[off:off + c]) if c else grouped.new_empty((0,)))
            off += c
        y = [o for o in outs if o.numel()]
        if y:
            import torch
            y_grouped = torch.cat(y, 0)
        else:
            y_grouped = grouped.new_empty((0,) + tuple(grouped.shape[1:]))
        return self.combine(y_grouped)

    def combine(self, y_grouped):
        import torch
        import torch.distributed as dist
        send, recv, perm = self._state
        dev = y_grouped.device
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm), dtype=np.int64)
        y_src = self.gather(y_grouped, torch.as_tensor(inv, device=dev)) if len(perm) else y_grouped
        back = y_grouped.new_empty((sum(send),) + tuple(y_grouped.shape[1:]))
        dist.all_to_all_single(back, y_src.contiguous(), send, recv)
        return back


class MoePlan:
    """qnb_moe_plan (include/qnb.h): the whole MoE forward as one device-driven call --
    trunk, gating, gate, routing, every expert on its device-resident sample count,
    combine and tail, captured as one CUDA graph (no host round trip)."""

    def __init__(self, net: "MoeNet", max_batch: int, use_cuda_graph: bool = True):
        lib = L.lib()
        parts = [net.trunk.layer_descs(), net.gating.layer_descs()]
        parts += [net.experts[e].layer_descs() for e in range(net.n_experts)]
        parts.append(net.tail.layer_descs())
        keep = []

        def gdesc(part):
            descs, n_blobs, k, _ = part
            arr = (L.LayerDesc * len(descs))(*descs)
            keep.extend([arr, k])
            return L.GraphDesc(arr, len(descs), n_blobs)

        gd = [gdesc(p) for p in parts]
        trunk, gating, tail = gd[0], gd[1], gd[-1]
        experts = (L.GraphDesc * net.n_experts)(*gd[2:-1])
        ml = net.moe_layer
        tb = G.infer_blobs(net.graph)
        bottom, top = ml["bottom"][0], ml["top"][0]
        in_dt = G.DTYPE_CODE[ml["bottom_data_type"]]
        top_dt = G.DTYPE_CODE[ml["top_data_type"]]
        qv_in = net.trunk.blob_qvals(bottom)
        qv_top = net.tail.blob_qvals(top)
        if in_dt in (2, 3) and qv_in is None:
            raise QnbError(5, "quantizer not finalized: " + bottom)
        if top_dt in (2, 3) and qv_top is None:
            raise QnbError(5, "quantizer not finalized: " + top)
        for k in ("gate_a", "gate_b", "gate_c"):
            if k not in net.gates:
                raise QnbError(1, f"missing parameter: {net.moe_name}.{k}")
        gsink = G.sinks(ml["moe"]["gating"])[-1]
        D = int(G.infer_blobs(ml["moe"]["gating"])[gsink]["shape"][1])
        if net.gates["gate_a"].shape != (net.n_experts, D):
            raise QnbError(2, "dimension mismatch")
        ga, gb, gc = (np.ascontiguousarray(net.gates[k], np.float32) for k in ("gate_a", "gate_b", "gate_c"))
        o = L.MoeOpts()
        o.max_batch, o.n_experts, o.top_k = max_batch, net.n_experts, net.top_k
        o.noise_enabled, o.seed, o.sample_offset = 1 if net.noise else 0, net.seed, 0
        o.in_dtype, o.top_dtype = in_dt, top_dt
        if qv_in is not None:
            o.in_qv = QVals(*qv_in.as_tuple())
        if qv_top is not None:
            o.top_qv = QVals(*qv_top.as_tuple())
        o.in_per_sample = int(np.prod(tb[bottom]["shape"][1:]))
        o.out_per_sample = int(np.prod(tb[top]["shape"][1:]))
        o.gate_dim = D
        o.gate_a, o.gate_b, o.gate_c = ga.ctypes.data, gb.ctypes.data, gc.ctypes.data
        o.use_cuda_graph = 1 if use_cuda_graph else 0
        self.max_batch, self.n_experts = max_batch, net.n_experts
        self.out_per_sample, self.top_dtype = o.out_per_sample, top_dt
        self.h = C.c_void_p()
        check(lib.qnb_moe_plan_create(C.byref(trunk), C.byref(gating), experts, C.byref(tail), C.byref(o),
                                      C.byref(self.h)))
        del keep

    def forward(self, x_ptr: int, out_ptr: int, batch: int, stream: int = 0, in_host: bool = False,
                out_host: bool = False) -> None:
        check(L.lib().qnb_moe_plan_forward(self.h, C.c_void_p(x_ptr), batch, 1 if in_host else 0,
                                           C.c_void_p(out_ptr), 1 if out_host else 0, C.c_void_p(stream)))

    def status(self, stream: int = 0) -> np.ndarray:
        """Synchronises; per-expert pair counts of the last forward (raises on degenerate gating)."""
        counts = (C.c_int64 * self.n_experts)()
        check(L.lib().qnb_moe_plan_status(self.h, counts, C.c_void_p(stream)))
        return np.array(counts[:], np.int64)

    def moe_output(self, batch: int) -> np.ndarray:
        ptr = C.c_void_p()
        check(L.lib().qnb_moe_plan_moe_output(self.h, C.byref(ptr)))
        dt = NP_OF[self.top_dtype]
        out = np.empty((batch, self.out_per_sample), dt)
        check(L.lib().qnb_memcpy_d2h(out.ctypes.data_as(C.c_void_p), ptr, out.nbytes, None))
        check(L.lib().qnb_stream_sync(None))
        return out

    def kernels_per_forward(self) -> int:
        k = C.c_int64()
        check(L.lib().qnb_moe_plan_stats(self.h, C.byref(k)))
        return k.value

    def __del__(self):
        try:
            if self.h:
                L.lib().qnb_moe_plan_destroy(self.h)
        except Exception:
            pass


class MoeNet:
    """qnet::Net surface for a graph with one MOE layer, backed by B200 plans.  One rank:
    the C-ABI MoE plan (MoePlan, device-driven, one CUDA graph).  N ranks: per-expert
    plans on this rank's experts with the expert all-to-all over torch.distributed."""

    BUCKET = 32

    def __init__(self, graph: dict, rank: int = 0, world: int = 1):
        self.graph = G.normalized(graph)
        trunk, moe, tail = split_moe_graph(self.graph)
        spec = moe["moe"]
        self.moe_name = moe["name"]
        self.n_experts, self.top_k = int(spec["n_experts"]), int(spec["top_k"])
        self.noise, self.seed = bool(spec.get("noise_enabled", False)), int(spec.get("seed", 0))
        self.moe_layer = moe
        self.trunk, self.tail = Net(trunk), Net(tail)
        self.gating = Net(spec["gating"])
        self.rank, self.world = rank, world
        self.per_rank = self.n_experts // world
        # every rank holds the parameters of all experts (set_param API), plans only for its own
        self.experts = [Net(spec["expert"]) for _ in range(self.n_experts)]
        self.gates = {}
        self.trunk_layers = {l["name"] for l in trunk["layers"]}
        self._pipes = {}
        self._mplans = {}
        self._last = None

    # ---- parameters / ranges (dotted names, src/net.cpp:161-204)
    def _route(self, name: str):
        m = _NESTED.match(name)
        if m and m.group(1) == self.moe_name:
            if m.group(2) == "gating":
                return self.gating, m.group(4)
            return self.experts[int(m.group(3))], m.group(4)
        return None, name

    def set_param(self, name, arr, dtype=0, qv=None):
        if name in (f"{self.moe_name}.gate_a", f"{self.moe_name}.gate_b", f"{self.moe_name}.gate_c"):
            self.gates[name.rsplit(".", 1)[1]] = np.ascontiguousarray(arr, np.float32)
            self._mplans.clear()
            return
        net, local = self._route(name)
        if net is None:
            net = self.trunk if name.split(".")[0] in self.trunk_layers else self.tail
        net.set_param(local, arr, dtype, qv)
        self._pipes.clear()
        self._mplans.clear()

    def set_range(self, key, lo, hi):
        net, local = self._route(key)
        if net is not None:
            net.set_range(local, lo, hi)
        else:
            self.trunk.set_range(key, lo, hi)
            self.tail.set_range(key, lo, hi)
        self._pipes.clear()
        self._mplans.clear()

    def finalize_quantizers(self):
        for n in [self.trunk, self.tail, self.gating] + self.experts:
            n.finalize_quantizers()
        self._pipes.clear()
        self._mplans.clear()

    def set_quant_mode(self, mode):
        for n in [self.trunk, self.tail, self.gating] + self.experts:
            n.set_quant_mode(mode)

    def blob_qvals(self, blob):
        return self.trunk.blob_qvals(blob) or self.tail.blob_qvals(blob)

    # ---- device pipeline
    def _pipe(self, B: int):
        if B in self._pipes:
            return self._pipes[B]
        import torch
        for k in ("gate_a", "gate_b", "gate_c"):
            if k not in self.gates:
                raise QnbError(1, f"missing parameter: {self.moe_name}.{k}")
        bottom = self.moe_layer["bottom"][0]
        tb = G.infer_blobs(self.graph)
        in_shape = tb[bottom]["shape"]
        qv_in = self.trunk.blob_qvals(bottom)
        if self.moe_layer["bottom_data_type"] in G.QUANT and qv_in is None:
            raise QnbError(5, "quantizer not finalized: " + bottom)
        top = self.moe_layer["top"][0]
        qv_top = self.tail.blob_qvals(top)
        gsink = G.sinks(self.moe_layer["moe"]["gating"])[-1]
        D = int(G.infer_blobs(self.moe_layer["moe"]["gating"])[gsink]["shape"][1])
        if self.gates["gate_a"].shape != (self.n_experts, D):
            raise QnbError(2, "dimension mismatch")
        per = int(np.prod(tb[top]["shape"][1:]))
        row_elems = int(np.prod(in_shape[1:]))
        cap = B * self.world  # an expert sees at most one pair per sample of every rank
        p = {
            "trunk": self.trunk.compile(B),
            "gating": self.gating.compile(B),
            "tail": self.tail.compile(B),
            # expert plans replay CUDA graphs at bucketed batch sizes (multiples of 32)
            "experts": {e: self.experts[e].compile(cap, use_cuda_graph=True)
                        for e in range(self.rank * self.per_rank, (self.rank + 1) * self.per_rank)},
            "D": D, "per": per, "row_elems": row_elems, "in_shape": in_shape,
            "in_dtype": G.DTYPE_CODE[self.moe_layer["bottom_data_type"]],
            "top_dtype": G.DTYPE_CODE[self.moe_layer["top_data_type"]],
            "qv_in": qv_in, "qv_top": qv_top,
        }
        dev = torch.device("cuda", torch.cuda.current_device())
        es = NP_OF[p["in_dtype"]]().itemsize
        P = B * self.top_k
        p["bufs"] = {
            "T": torch.empty(B * row_elems * es, dtype=torch.uint8, device=dev),
            "F": torch.empty(B * row_elems, dtype=torch.float32, device=dev),
            "feats": torch.empty(B * D, dtype=torch.float32, device=dev),
            "idx": torch.empty(P, dtype=torch.int64, device=dev),
            "w": torch.empty(P, dtype=torch.float32, device=dev),
            "counts": torch.empty(self.n_experts, dtype=torch.int64, device=dev),
            "pair_sample": torch.empty(max(P, self.n_experts * (cap + self.BUCKET)), dtype=torch.int64, device=dev),
            "pair_slot": torch.empty(P, dtype=torch.int64, device=dev),
            "S": torch.empty((max(P, self.n_experts * (cap + self.BUCKET)), row_elems * es), dtype=torch.uint8,
                             device=dev),
            # + kBucket rows: an expert's bucketed batch may run past its segment (read-only
            # spill into the next expert's rows, whose outputs are written after it)
            "X": torch.empty((self.per_rank * (cap + self.BUCKET)) * row_elems, dtype=torch.float32, device=dev),
            "Y": torch.empty((self.per_rank * (cap + self.BUCKET), per), dtype=torch.float32, device=dev),
            "M": torch.empty(B * per * NP_OF[p["top_dtype"]]().itemsize, dtype=torch.uint8, device=dev),
            "wa": torch.from_numpy(self.gates["gate_a"]).to(dev),
            "wb": torch.from_numpy(self.gates["gate_b"]).to(dev),
            "wc": torch.from_numpy(self.gates["gate_c"]).to(dev),
        }
        if self.world > 1:
            lib = L.lib()

            def gather(t, rows):
                out = t.new_empty((rows.numel(),) + tuple(t.shape[1:]))
                rb = t[0].numel() * t.element_size() if t.shape[0] else 0
                check(lib.qnb_gather_rows(t.data_ptr(), rb, rows.data_ptr(), rows.numel(), out.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
                return out
            p["xchg"] = ExpertExchange(self.n_experts, self.rank, self.world, gather)
        self._pipes[B] = p
        return p

    def moe_plan(self, B: int) -> MoePlan:
        if B not in self._mplans:
            self._mplans[B] = MoePlan(self, B)
        return self._mplans[B]

    @property
    def last_stats(self) -> dict:
        """Routing statistics of the last forward (synchronises on the MoE plan path)."""
        if self._last is None:
            return {"counts": np.zeros(self.n_experts, np.int64)}
        if isinstance(self._last, MoePlan):
            import torch
            return {"counts": self._last.status(torch.cuda.current_stream().cuda_stream)}
        return self._last

    def moe_output(self, B: int) -> np.ndarray:
        """The MoE layer's top blob of the last forward at batch B, (B, features) in the
        top dtype (a checkpoint for parity tests)."""
        if self.world == 1:
            return self.moe_plan(B).moe_output(B)
        p = self._pipes[B]
        return p["bufs"]["M"].cpu().numpy().view(NP_OF[p["top_dtype"]]).reshape(B, p["per"])

    def forward_device(self, x_ptr: int, out_ptr: int, B: int, in_host: bool = False,
                       out_host: bool = False):
        """One MoE forward on torch's current stream (device buffers, or pinned host
        buffers).  One rank: the device-driven MoE plan, nothing returns to the host."""
        if self.world == 1:
            import torch
            mp = self.moe_plan(B)
            mp.forward(x_ptr, out_ptr, B, torch.cuda.current_stream().cuda_stream, in_host, out_host)
            self._last = mp
            return None
        return self._forward_device_xchg(x_ptr, out_ptr, B, in_host, out_host)

    def _forward_device_xchg(self, x_ptr: int, out_ptr: int, B: int, in_host: bool = False,
                             out_host: bool = False) -> dict:
        """One MoE forward (stream: torch's current stream) on device buffers, or on pinned
        host buffers: the trunk plan then pipelines the input's H2D copy chunk by chunk
        under its own compute, and the tail plan copies the result back.  Returns routing
        statistics (per-expert counts) for load-balance reporting."""
        import torch
        p = self._pipe(B)
        b = p["bufs"]
        lib = L.lib()
        s = torch.cuda.current_stream().cuda_stream
        sp = C.c_void_p(s)
        n = B * p["row_elems"]
        p["trunk"].forward_device(x_ptr, b["T"].data_ptr(), B, s, in_host=in_host)
        if p["qv_in"] is not None:
            check(lib.qnb_dequantize(b["T"].data_ptr(), n, p["in_dtype"], C.byref(p["qv_in"]), b["F"].data_ptr(),
                                     sp))
        else:
            check(lib.qnb_cast_float(b["T"].data_ptr(), n, p["in_dtype"], L.FP32, b["F"].data_ptr(), sp))
        p["gating"].forward_device(b["F"].data_ptr(), b["feats"].data_ptr(), B, s)
        # the gating noise is keyed on the global sample index (rank r holds rows r*B..)
        check(lib.qnb_moe_gate_at(b["feats"].data_ptr(), B, p["D"], b["wa"].data_ptr(), b["wb"].data_ptr(),
                                  b["wc"].data_ptr(), self.n_experts, self.top_k, 1 if self.noise else 0,
                                  C.c_uint64(self.seed), self.rank * B, b["idx"].data_ptr(), b["w"].data_ptr(), sp))
        # dense per-expert rows; the all-to-all splits count real pairs
        check(lib.qnb_moe_route(b["idx"].data_ptr(), B, self.top_k, self.n_experts, 0, b["counts"].data_ptr(),
                                b["pair_sample"].data_ptr(), b["pair_slot"].data_ptr(), sp))
        P = B * self.top_k
        es = b["S"].shape[1] // p["row_elems"]
        check(lib.qnb_gather_rows(b["T"].data_ptr(), p["row_elems"] * es, b["pair_sample"].data_ptr(), P,
                                  b["S"].data_ptr(), sp))
        counts = b["counts"].cpu().numpy()  # the all-to-all needs the split sizes on the host
        xoff = [0]

        def expert_fn(e, rows_e):
            """Expert e (a local plan) on the rows it received: dequantize -> plan -> FP32."""
            c = rows_e.shape[0]
            x_dst = b["X"].data_ptr() + xoff[0] * p["row_elems"] * 4
            ne = c * p["row_elems"]
            if p["qv_in"] is not None:
                check(lib.qnb_dequantize(rows_e.data_ptr(), ne, p["in_dtype"], C.byref(p["qv_in"]), x_dst, sp))
            else:
                check(lib.qnb_cast_float(rows_e.data_ptr(), ne, p["in_dtype"], L.FP32, x_dst, sp))
            y = b["Y"][xoff[0]:xoff[0] + c]
            p["experts"][e].forward_device(x_dst, y.data_ptr(), c, s)
            xoff[0] += c
            return y

        y = p["xchg"].run(b["S"][:P], counts, expert_fn)
        qv = C.byref(p["qv_top"]) if p["qv_top"] is not None else None
        check(lib.qnb_moe_combine_rows(y.data_ptr(), p["per"], b["pair_slot"].data_ptr(), b["w"].data_ptr(), B,
                                       self.top_k, p["top_dtype"], qv, b["M"].data_ptr(), sp))
        p["tail"].forward_device(b["M"].data_ptr(), out_ptr, B, s, out_host=out_host)
        self._last = {"counts": counts}
        return self._last

    def forward(self, inputs: dict) -> dict:
        """Net::forward (src/net.cpp:305-330) with host arrays in and out."""
        import torch
        name = G.input_name(self.graph)
        if name not in inputs:
            raise QnbError(1, "missing input: " + name)
        x = np.ascontiguousarray(inputs[name])
        B = x.shape[0]
        sink = G.sinks(self.graph)[-1]
        info = G.infer_blobs(self.graph)[sink]
        xd = torch.from_numpy(x).cuda()
        out = np.empty((B,) + tuple(info["shape"][1:]), NP_OF[G.DTYPE_CODE[info["dtype"]]])
        od = torch.empty(out.nbytes, dtype=torch.uint8, device="cuda")
        self.forward_device(xd.data_ptr(), od.data_ptr(), B)
        out[...] = od.cpu().numpy().view(out.dtype).reshape(out.shape)
        return {G.sinks(self.graph)[-1]: out}


__all__ = ["MoeNet", "MoePlan", "ExpertExchange", "split_moe_graph", "QUANTIZED", "QVals"]
