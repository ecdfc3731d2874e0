"""Host graph logic the plan compiler needs, restated from the reference:

  override_precision   src/graph.cpp:343-406  retype layers, insert QUANTIZER layers
  infer_blobs          src/graph.cpp:247-318  blob dtype / shape / producer / consumers
  range_key            src/net.cpp:66-73, 85-94  calibration-range aliasing

tests/test_graph.py checks these against the compiled reference (graph_to_json of
override_precision, Net ranges) on every model fixture.
"""
from __future__ import annotations

import copy

import numpy as np

FP32, FP16, INT8Q, INT16Q = "fp32", "fp16", "int8", "int16"
QUANT = (INT8Q, INT16Q)
FLOAT = (FP32, FP16)
KIND_CODE = {"input": 0, "conv": 1, "pool": 2, "inner_product": 3, "relu": 4, "lrn": 5, "softmax": 6,
             "quantizer": 7, "dropout": 8, "moe": 9}
DTYPE_CODE = {FP32: 0, FP16: 1, INT8Q: 2, INT16Q: 3}


def _types(l):
    mi = l.get("bottom_data_type", FP32)
    d = l.get("compute_data_type", mi)
    mo = l.get("top_data_type", d)
    return mi, d, mo


def normalized(g: dict) -> dict:
    """Graph with explicit bottom/compute/top data types on every layer (the JSON
    defaults of src/graph_json.cpp:48-50)."""
    g = copy.deepcopy(g)
    for l in g["layers"]:
        mi, d, mo = _types(l)
        l["bottom_data_type"], l["compute_data_type"], l["top_data_type"] = mi, d, mo
    return g


def override_precision(g: dict, target: str) -> dict:
    """src/graph.cpp:343-406."""
    g = normalized(g)
    out = {"name": g.get("name", ""), "layers": [], "inspect": list(g.get("inspect", [])),
           "range_aliases": dict(g.get("range_aliases", {}))}
    staged = copy.deepcopy(g["layers"])
    for l in staged:
        k = l["kind"]
        if k == "input":
            continue
        if k in ("softmax", "lrn"):
            l["bottom_data_type"] = l["compute_data_type"] = l["top_data_type"] = FP32
        elif k == "quantizer":
            if l["top_data_type"] not in FLOAT:
                l["top_data_type"] = target
        else:
            l["bottom_data_type"] = l["compute_data_type"] = l["top_data_type"] = target

    def root(b):
        seen = set()
        while b in out["range_aliases"] and b not in seen:
            seen.add(b)
            b = out["range_aliases"][b]
        return b

    blob_type = {}
    converted = {}
    for l in staged:
        if l["kind"] == "input":
            blob_type[l["top"][0]] = l["top_data_type"]
            out["layers"].append(l)
            continue
        b = l["bottom"][0]
        have = blob_type[b]
        if l["kind"] == "quantizer":
            l["bottom_data_type"] = l["compute_data_type"] = have
        elif l["bottom_data_type"] != have:
            key = (b, l["bottom_data_type"])
            if key not in converted:
                q = {"name": f"{b}_to_{l['bottom_data_type']}", "kind": "quantizer",
                     "bottom_data_type": have, "compute_data_type": have,
                     "top_data_type": l["bottom_data_type"], "bottom": [b],
                     "top": [f"{b}__{l['bottom_data_type']}"]}
                blob_type[q["top"][0]] = q["top_data_type"]
                out["range_aliases"][q["top"][0]] = root(b)
                out["layers"].append(q)
                converted[key] = q["top"][0]
            l["bottom"] = [converted[key]]
        blob_type[l["top"][0]] = l["top_data_type"]
        out["layers"].append(l)
    return out


def infer_blobs(g: dict, batch: int | None = None) -> dict:
    """blob -> {dtype, shape, producer, consumers}  (src/graph.cpp:247-318)."""
    g = normalized(g)
    blobs = {}
    for i, l in enumerate(g["layers"]):
        for b in l.get("bottom", []):
            blobs[b]["consumers"].append(i)
        k = l["kind"]
        if k == "input":
            shape = list(l["input_shape"])
            if batch is not None:
                shape[0] = batch
        else:
            ins = blobs[l["bottom"][0]]["shape"]
            if k == "conv":
                c = l["conv"]
                oh = (ins[2] + 2 * c.get("pad_h", 0) - c["kernel_h"]) // c.get("stride_h", 1) + 1
                ow = (ins[3] + 2 * c.get("pad_w", 0) - c["kernel_w"]) // c.get("stride_w", 1) + 1
                shape = [ins[0], c["out_channels"], oh, ow]
            elif k == "pool":
                p = l["pool"]
                shape = [ins[0], ins[1], (ins[2] - p["kernel"]) // p["stride"] + 1,
                         (ins[3] - p["kernel"]) // p["stride"] + 1]
            elif k == "inner_product":
                shape = [ins[0], l["num_output"]]
            elif k == "moe":
                sub = infer_blobs(l["moe"]["expert"])
                sink = [v for v in sub.values() if not v["consumers"]][-1]
                shape = [ins[0]] + list(sink["shape"][1:])
            else:
                shape = list(ins)
        blobs[l["top"][0]] = {"dtype": l["top_data_type"], "shape": shape, "producer": i, "consumers": []}
    return blobs


def range_aliases(g: dict) -> dict:
    """Net's alias table: graph range_aliases plus POOL / DROPOUT tops aliasing their
    bottoms (src/net.cpp:66-73)."""
    al = dict(g.get("range_aliases", {}))

    def resolve(b):
        hops = 0
        while b in al and hops < 1024:
            b = al[b]
            hops += 1
        return b

    for l in g["layers"]:
        if l["kind"] in ("pool", "dropout"):
            al[l["top"][0]] = resolve(l["bottom"][0])
    return al


def range_key(aliases: dict, blob: str) -> str:
    hops = 0
    while blob in aliases and hops < 1024:
        blob = aliases[blob]
        hops += 1
    return blob


def sinks(g: dict) -> list:
    blobs = infer_blobs(g)
    return sorted([b for b, v in blobs.items() if not v["consumers"]], key=lambda b: blobs[b]["producer"])


def input_name(g: dict) -> str:
    for l in g["layers"]:
        if l["kind"] == "input":
            return l["top"][0]
    raise ValueError("missing input")


def conv_flops(g: dict, batch: int) -> dict:
    """Algorithmic operations (2 per MAC) per conv / inner-product layer."""
    blobs = infer_blobs(g, batch)
    out = {}
    for l in normalized(g)["layers"]:
        if l["kind"] == "conv":
            c = l["conv"]
            ins, o = blobs[l["bottom"][0]]["shape"], blobs[l["top"][0]]["shape"]
            K = ins[1] // c.get("groups", 1) * c["kernel_h"] * c["kernel_w"]
            out[l["name"]] = 2 * o[0] * o[1] * o[2] * o[3] * K
        elif l["kind"] == "inner_product":
            ins = blobs[l["bottom"][0]]["shape"]
            out[l["name"]] = 2 * ins[0] * int(np.prod(ins[1:])) * l["num_output"]
    return out
