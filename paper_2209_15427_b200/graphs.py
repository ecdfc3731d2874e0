"""Model fixtures in the reference's graph-JSON schema (src/graph_json.cpp:31-141).

The reference ships only a one-neuron graph (graphs/celsius.json); the benchmark
models are authored here: AlexNet in CaffeNet order
(PAPER.md:855-868), AlexNet-MoE, VGG-16 and LeNet-5.  The same
JSON text is consumed by the reference (graph_from_json) and by our plan compiler,
so both sides run literally the same graph.

Parameters use the reference's layouts: conv weights OC x C/g x KH x KW, inner
product weights K x OUT (README.md:179-180), FP32 biases.  Synthetic values are
seeded: weights U(-1/sqrt(fan_in), 1/sqrt(fan_in)), biases U(-0.1, 0.1),
images U(0, 255).
"""
from __future__ import annotations

import copy
import json

import numpy as np


def _input(name, shape):
    return {"name": name, "kind": "input", "top": [name], "input_shape": list(shape)}


def _conv(name, bottom, out, k, s=1, p=0, g=1, top=None):
    return {"name": name, "kind": "conv", "bottom": [bottom], "top": [top or name],
            "conv": {"out_channels": out, "kernel_h": k, "kernel_w": k, "stride_h": s, "stride_w": s,
                     "pad_h": p, "pad_w": p, "groups": g, "bias_term": True}}


def _relu(name, blob):
    return {"name": name, "kind": "relu", "bottom": [blob], "top": [name]}


def _pool(name, bottom, k, s):
    return {"name": name, "kind": "pool", "bottom": [bottom], "top": [name], "pool": {"kernel": k, "stride": s}}


def _lrn(name, bottom):
    return {"name": name, "kind": "lrn", "bottom": [bottom], "top": [name],
            "lrn": {"local_size": 5, "alpha": 1e-4, "beta": 0.75, "k": 1.0}}


def _ip(name, bottom, out):
    return {"name": name, "kind": "inner_product", "bottom": [bottom], "top": [name], "num_output": out,
            "bias_term": True}


def _drop(name, bottom):
    return {"name": name, "kind": "dropout", "bottom": [bottom], "top": [name]}


def _softmax(name, bottom):
    return {"name": name, "kind": "softmax", "bottom": [bottom], "top": [name]}


def alexnet(batch: int = 1) -> dict:
    """AlexNet / CaffeNet, 3x227x227 input, 1000 classes."""
    L = [
        _input("data", [batch, 3, 227, 227]),
        _conv("conv1", "data", 96, 11, s=4), _relu("relu1", "conv1"), _pool("pool1", "relu1", 3, 2),
        _lrn("norm1", "pool1"),
        _conv("conv2", "norm1", 256, 5, p=2, g=2), _relu("relu2", "conv2"), _pool("pool2", "relu2", 3, 2),
        _lrn("norm2", "pool2"),
        _conv("conv3", "norm2", 384, 3, p=1), _relu("relu3", "conv3"),
        _conv("conv4", "relu3", 384, 3, p=1, g=2), _relu("relu4", "conv4"),
        _conv("conv5", "relu4", 256, 3, p=1, g=2), _relu("relu5", "conv5"), _pool("pool5", "relu5", 3, 2),
        _ip("fc6", "pool5", 4096), _relu("relu6", "fc6"), _drop("drop6", "relu6"),
        _ip("fc7", "drop6", 4096), _relu("relu7", "fc7"), _drop("drop7", "relu7"),
        _ip("fc8", "drop7", 1000), _softmax("prob", "fc8"),
    ]
    return {"name": "alexnet", "layers": L}


def vgg16(batch: int = 1, res: int = 224) -> dict:
    """VGG-16 (configuration D), 3 x res x res input (224 for the benchmark; the
    parity tests use res=32, which keeps every layer kind and shape rule)."""
    L = [_input("data", [batch, 3, res, res])]
    cur = "data"
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]
    blk, idx = 1, 1
    for v in cfg:
        if v == "M":
            L.append(_pool(f"pool{blk}", cur, 2, 2))
            cur = f"pool{blk}"
            blk, idx = blk + 1, 1
            continue
        name = f"conv{blk}_{idx}"
        L.append(_conv(name, cur, v, 3, p=1))
        L.append(_relu(f"relu{blk}_{idx}", name))
        cur = f"relu{blk}_{idx}"
        idx += 1
    L += [_ip("fc6", cur, 4096), _relu("relu6", "fc6"), _drop("drop6", "relu6"),
          _ip("fc7", "drop6", 4096), _relu("relu7", "fc7"), _drop("drop7", "relu7"),
          _ip("fc8", "drop7", 1000), _softmax("prob", "fc8")]
    return {"name": "vgg16", "layers": L}


def lenet5(batch: int = 1) -> dict:
    """LeNet-5 (Caffe variant): conv20 k5, pool, conv50 k5, pool, ip500, relu, ip10."""
    L = [
        _input("data", [batch, 1, 28, 28]),
        _conv("conv1", "data", 20, 5), _pool("pool1", "conv1", 2, 2),
        _conv("conv2", "pool1", 50, 5), _pool("pool2", "conv2", 2, 2),
        _ip("ip1", "pool2", 500), _relu("relu1", "ip1"), _ip("ip2", "relu1", 10),
    ]
    return {"name": "lenet5", "layers": L}


def _quantizer(name, bottom, top_type):
    return {"name": name, "kind": "quantizer", "bottom": [bottom], "top": [name], "top_data_type": top_type}


def alexnet_moe(batch: int = 1, dtype: str = "int8", n_experts: int = 16, top_k: int = 4) -> dict:
    """AlexNet-MoE.  override_precision does not recurse into the
    nested graphs (src/graph.cpp:351-368), so the sub-graphs are typed explicitly and
    end in a ->fp32 quantizer (moe_forward needs FP32 features, src/moe.cpp:178-181)."""
    def typed(layers, t):
        out = []
        for l in layers:
            l = copy.deepcopy(l)
            if l["kind"] in ("conv", "relu", "pool", "inner_product", "dropout"):
                l["bottom_data_type"] = l["compute_data_type"] = l["top_data_type"] = t
            out.append(l)
        return out

    def sub(name, body_fn):
        # input FP32 (48 x 27 x 27 dequantized trunk features), then t-typed body
        L = [_input("x", [1, 48, 27, 27]), _quantizer("x_to_q", "x", dtype)]
        L[1]["bottom_data_type"] = "fp32"
        L[1]["compute_data_type"] = "fp32"
        body = body_fn("x_to_q")
        L += typed(body[:-1], dtype)
        tail = body[-1]
        L.append(tail)
        return {"name": name, "layers": L}

    def lrn_q(name, bottom):
        # LRN is FP32-only (src/graph.cpp:208-213): bracket it with quantizers
        to_f, to_q = _quantizer(f"{bottom}_f", bottom, "fp32"), _quantizer(f"{name}_q", name, dtype)
        to_f["bottom_data_type"] = to_f["compute_data_type"] = dtype  # quantizers compute at d = mi
        to_q["bottom_data_type"] = to_q["compute_data_type"] = "fp32"
        return [to_f, _lrn(name, f"{bottom}_f"), to_q]

    def gating_body(x):
        L = [_conv("g_conv", x, 64, 5, p=2, g=2), _relu("g_relu", "g_conv"), _pool("g_pool", "g_relu", 3, 2)]
        L += lrn_q("g_norm", "g_pool")
        L += [_ip("g_fc1", "g_norm_q", 128), _relu("g_relu2", "g_fc1"), _ip("g_fc2", "g_relu2", n_experts)]
        L.append(_quantizer("feats", "g_fc2", "fp32"))
        return L

    def expert_body(x):
        L = [_conv("e_conv1", x, 64, 5, p=2, g=2), _relu("e_relu1", "e_conv1"), _pool("e_pool1", "e_relu1", 3, 2)]
        L += lrn_q("e_norm1", "e_pool1")
        L += [_conv("e_conv2", "e_norm1_q", 96, 3, p=1), _relu("e_relu2", "e_conv2"),
              _conv("e_conv3", "e_relu2", 96, 3, p=1, g=2), _relu("e_relu3", "e_conv3"),
              _conv("e_conv4", "e_relu3", 64, 3, p=1, g=2), _relu("e_relu4", "e_conv4"),
              _pool("e_pool2", "e_relu4", 3, 2),
              _ip("e_fc1", "e_pool2", 1024), _relu("e_relu5", "e_fc1"), _drop("e_drop", "e_relu5"),
              _ip("e_fc2", "e_drop", 2048)]
        L.append(_quantizer("y", "e_fc2", "fp32"))
        return L

    gating = sub("gating", gating_body)
    expert = sub("expert", expert_body)
    for g in (gating, expert):  # the quantizer tails compute at the body type
        g["layers"][-1]["bottom_data_type"] = dtype
        g["layers"][-1]["compute_data_type"] = dtype
    L = [
        _input("data", [batch, 3, 227, 227]),
        _conv("conv1", "data", 48, 11, s=4), _relu("relu1", "conv1"), _pool("pool1", "relu1", 3, 2),
        _lrn("norm1", "pool1"),
        {"name": "moe", "kind": "moe", "bottom": ["norm1"], "top": ["moe"],
         "moe": {"n_experts": n_experts, "top_k": top_k, "batch_mode": "all_experts", "noise_enabled": False,
                 "seed": 0, "gating": gating, "expert": expert}},
        _relu("relu_moe", "moe"), _drop("drop_moe", "relu_moe"),
        _ip("fc", "drop_moe", 1000), _softmax("prob", "fc"),
    ]
    return {"name": "alexnet_moe", "layers": L}


def conv_layer(batch: int = 128, channels: int = 64, res: int = 56, out_channels: int = 64, k: int = 3,
               stride: int = 1, pad: int = -1) -> dict:
    """One convolution (BASELINE configs[4]: the single conv-layer sweep, C/K 64-512,
    3x3/5x5/11x11, stride 1/2/4 at 56x56).  pad defaults to k // 2."""
    p = k // 2 if pad < 0 else pad
    L = [_input("data", [batch, channels, res, res]), _conv("conv", "data", out_channels, k, stride, p)]
    return {"name": f"conv_c{channels}_k{out_channels}_r{k}_s{stride}", "layers": L}


MODELS = {"alexnet": alexnet, "vgg16": vgg16, "lenet5": lenet5,
          "vgg16_32": lambda batch=1: vgg16(batch, res=32)}


def to_json(g: dict) -> str:
    return json.dumps(g)


# ------------------------------------------------------------- parameters
def param_specs(g: dict, shapes: dict):
    """[(name, shape, fan_in)] for conv / inner-product layers, in layer order.
    `shapes` maps blob -> shape (from graph.infer_blobs)."""
    out = []
    for l in g["layers"]:
        if l["kind"] == "conv":
            c = l["conv"]
            cin = shapes[l["bottom"][0]][1]
            fan = cin // c.get("groups", 1) * c["kernel_h"] * c["kernel_w"]
            out.append((l["name"] + ".weight", (c["out_channels"], cin // c.get("groups", 1), c["kernel_h"],
                                                 c["kernel_w"]), fan))
            out.append((l["name"] + ".bias", (c["out_channels"],), None))
        elif l["kind"] == "inner_product":
            shp = shapes[l["bottom"][0]]
            K = int(np.prod(shp[1:]))
            out.append((l["name"] + ".weight", (K, l["num_output"]), K))
            out.append((l["name"] + ".bias", (l["num_output"],), None))
    return out


def synth_params(g: dict, shapes: dict, seed: int = 20261017) -> dict:
    """Seeded synthetic FP32 parameters, one generator per parameter in layer order."""
    params = {}
    for i, (name, shape, fan) in enumerate(param_specs(g, shapes)):
        rng = np.random.default_rng(seed + 7919 * (i + 1))
        if fan is None:
            params[name] = rng.uniform(-0.1, 0.1, shape).astype(np.float32)
        else:
            b = 1.0 / np.sqrt(fan)
            params[name] = rng.uniform(-b, b, shape).astype(np.float32)
    return params


def synth_images(n: int, shape, seed: int = 20261017, offset: int = 0) -> np.ndarray:
    """U(0, 255) FP32 images, image i from its own seeded generator."""
    out = np.empty((n,) + tuple(shape), np.float32)
    for i in range(n):
        out[i] = np.random.default_rng(seed + offset + i).uniform(0.0, 255.0, shape).astype(np.float32)
    return out


def moe_layer(g: dict) -> dict:
    return next(l for l in g["layers"] if l["kind"] == "moe")


def synth_params_moe(g: dict, seed: int = 20261017) -> dict:
    """Seeded parameters of an MoE graph under the reference's dotted names
    (include/qnet/net.hpp:36-40): trunk/tail layers by name, "<moe>.gating.<p>",
    "<moe>.expert<k>.<p>", and the gate matrices "<moe>.gate_a/_b/_c" with
    W_a ~ U(-0.5, 0.5), W_b = W_c = 0 (noise off)."""
    from . import graph as G
    m = moe_layer(g)
    name, spec = m["name"], m["moe"]
    main = {"name": g.get("name", ""), "layers": [l for l in g["layers"] if l["kind"] != "moe"]}
    shapes = {}
    for b, v in G.infer_blobs(g).items():
        shapes[b] = v["shape"]
    params = {}
    # trunk and tail layers (the MoE layer owns no weight of its own besides the gates)
    specs = [s for s in param_specs(g, shapes)]
    for i, (pname, shape, fan) in enumerate(specs):
        rng = np.random.default_rng(seed + 7919 * (i + 1))
        b = 0.1 if fan is None else 1.0 / np.sqrt(fan)
        params[pname] = rng.uniform(-b, b, shape).astype(np.float32)
    del main
    gshapes = {b: v["shape"] for b, v in G.infer_blobs(spec["gating"]).items()}
    for k, v in synth_params(spec["gating"], gshapes, seed=seed + 1).items():
        params[f"{name}.gating.{k}"] = v
    eshapes = {b: v["shape"] for b, v in G.infer_blobs(spec["expert"]).items()}
    for e in range(spec["n_experts"]):
        for k, v in synth_params(spec["expert"], eshapes, seed=seed + 101 * (e + 2)).items():
            params[f"{name}.expert{e}.{k}"] = v
    D = [v for v in G.infer_blobs(spec["gating"]).values() if not v["consumers"]][-1]["shape"][1]
    N = spec["n_experts"]
    rng = np.random.default_rng(seed + 99991)
    params[f"{name}.gate_a"] = rng.uniform(-0.5, 0.5, (N, D)).astype(np.float32)
    params[f"{name}.gate_b"] = np.zeros((N, D), np.float32)
    params[f"{name}.gate_c"] = np.zeros((N,), np.float32)
    return params


MODELS["alexnet_moe"] = alexnet_moe
