"""Generates the calibration fixtures (range per calibration key) with the UNMODIFIED
reference: qnet::Net in OBSERVE mode over seeded synthetic images
(calibrate on 8 separate seeded images; here `--images`), exactly as
`qnet observe` does (tools/qnet_main.cpp:144-161).

Both the B200 plan and the reference arm load these ranges with set_range(), so the
two run on identical integer grids.  Run in the build container (needs oracle/_ref):

    python tests/golden/make_calibration.py --model alexnet --precision int8 --images 4
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import ffi  # noqa: E402
from paper_2209_15427_b200 import graph as G  # noqa: E402
from paper_2209_15427_b200 import graphs  # noqa: E402

DT = {"fp32": 0, "fp16": 1, "int8": 2, "int16": 3}


def observe_one(args):
    model, precision, idx = args
    g = graphs.MODELS[model](1)
    ref = ffi.Reference()
    net = ref.net(json.dumps(g), DT[precision])
    rg = json.loads(net.graph_json())
    shapes = {b: v["shape"] for b, v in G.infer_blobs(g).items()}
    moe = [l for l in g["layers"] if l["kind"] == "moe"]
    params = graphs.synth_params_moe(g) if moe else graphs.synth_params(g, shapes)
    for name, arr in params.items():
        net.set_param(name, arr)
    net.set_mode(1)  # OBSERVE
    inp = G.input_name(g)
    x = graphs.synth_images(1, shapes[inp][1:], offset=1000 + idx)
    net.forward(inp, x)
    out = {}
    for b in G.infer_blobs(rg):
        r = net.range(b)
        if r is not None:
            out[G.range_key(G.range_aliases(rg), b)] = r
    for m in moe:  # nested nets: "<moe>.gating.<key>", "<moe>.expert<k>.<key>" (src/net.cpp:161-167)
        subs = [("gating", m["moe"]["gating"])] + [(f"expert{k}", m["moe"]["expert"])
                                                   for k in range(m["moe"]["n_experts"])]
        for prefix, sg in subs:
            al = G.range_aliases(G.normalized(sg))
            for b in G.infer_blobs(sg):
                key = G.range_key(al, b)
                r = net.range(f"{m['name']}.{prefix}.{key}")
                if r is not None:
                    out[f"{m['name']}.{prefix}.{key}"] = r
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="alexnet")
    ap.add_argument("--precision", default="int8")
    ap.add_argument("--images", type=int, default=4)
    a = ap.parse_args()
    t0 = time.time()
    with ProcessPoolExecutor(max_workers=min(a.images, os.cpu_count() or 1)) as ex:
        parts = list(ex.map(observe_one, [(a.model, a.precision, i) for i in range(a.images)]))
    ranges = {}
    for p in parts:  # observation only widens (include/qnet/quantizer_values.hpp:44-52)
        for k, (lo, hi) in p.items():
            if k in ranges:
                ranges[k] = (min(ranges[k][0], lo), max(ranges[k][1], hi))
            else:
                ranges[k] = (lo, hi)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{a.model}_{a.precision}_calib.json")
    with open(path, "w") as f:
        json.dump({"model": a.model, "precision": a.precision, "images": a.images,
                   "image_seed_offset": 1000, "ranges": ranges}, f, indent=1, sort_keys=True)
    print(f"wrote {path}: {len(ranges)} keys in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
