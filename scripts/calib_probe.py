"""Prints how far the device OBSERVE ranges / PSEUDO outputs are from the reference's."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import test_gpu_calibration as T
from paper_2209_15427_b200 import graph as G, graphs
from paper_2209_15427_b200.net import OBSERVE, PSEUDO

for model in ["lenet5", "vgg16_32", "alexnet"]:
    gold = T._golden(model)
    net, g, shapes = T._net(model)
    inp = G.input_name(g)
    x = graphs.synth_images(gold["images"], shapes[inp][1:], offset=gold["image_seed_offset"])
    net.set_quant_mode(OBSERVE)
    net.forward({inp: x})
    worst = max((max(abs(net.ranges[k][0] - lo), abs(net.ranges[k][1] - hi)) / max(abs(lo), abs(hi)), k)
                for k, (lo, hi) in gold["ranges"].items())
    exact = sum(1 for k, (lo, hi) in gold["ranges"].items() if tuple(net.ranges[k]) == (lo, hi))
    print(model, "observe worst rel", worst, "exact", exact, "/", len(gold["ranges"]))
    net, g, shapes = T._finalized(model)
    x = graphs.synth_images(2, shapes[inp][1:], offset=41)
    net.set_quant_mode(PSEUDO)
    (_, mine), = net.forward({inp: x}).items()
    theirs = T._ref_pseudo(model, x)
    d = np.abs(mine - theirs)
    print(model, "pseudo max abs", d.max(), "range", theirs.max() - theirs.min(), "n differ", int((d > 0).sum()), "/", d.size)
