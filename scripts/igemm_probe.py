"""Per-layer times of the AlexNet INT8 plan under the igemm profiling probes
(QNB_IGEMM_DBG: 1 = epilogue skips its math, 2 = no MMAs, 3 = both).  Prints one
JSON line per probe setting; run each setting in its own process."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2209_15427_b200 import graph as G, graphs
from paper_2209_15427_b200.net import QUANTIZED, Net
g, shapes, params, ranges = bench.model_setup("alexnet", "int8")
net = Net(G.override_precision(g, "int8"))
for k, v in params.items(): net.set_param(k, v)
for k, (lo, hi) in ranges.items(): net.set_range(k, lo, hi)
net.finalize_quantizers(); net.set_quant_mode(QUANTIZED)
B = 256
plan = net.compile(B)
x = torch.from_numpy(graphs.synth_images(B, shapes["data"][1:])).cuda()
o = torch.empty((B, 1000), device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    plan.forward_device(x.data_ptr(), o.data_ptr(), B, sp)
plan.profile(x.data_ptr(), o.data_ptr(), B, 3, sp)
ms = plan.profile(x.data_ptr(), o.data_ptr(), B, 10, sp)
names = [l["name"] for l in net.graph["layers"]]
print(json.dumps({"dbg": os.environ.get("QNB_IGEMM_DBG", "0"),
                  "steps": [(names[li], k, round(t * 1000, 1)) for (li, k, _, _), t in zip(plan.steps(), ms)]}))
