"""The drop-in from the reference's side: qnet::Net (unmodified reference, C++) vs
qnb::Executor (include/qnb_qnet.hpp over the C-ABI) on the same calibrated net.

tests/cpp/executor_check.cpp is compiled by oracle/Makefile (in the build container,
where /root/reference exists) into oracle/_ref/qnb_executor_check; the binary travels
to the GPU box with the snapshot.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "qnb_executor_check")
GRAPHS = os.path.join(ROOT, "tests", "golden", "graphs")


def run(graph, precision, batch, calib=1, timeout=900):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/qnb_executor_check not built (needs /root/reference at build time)")
    return subprocess.run([BIN, os.path.join(GRAPHS, graph + ".json"), precision, str(batch), str(calib)],
                          capture_output=True, text=True, timeout=timeout)


def test_executor_fails_loudly_without_gpu():
    """CPU: no silent fallback — the C++ executor throws the backend's CUDA error."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    r = run("lenet5", "int8", 2, timeout=120)
    assert r.returncode != 0
    assert "no CPU fallback" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("graph,precision,batch", [
    ("lenet5", "int8", 64),
    ("lenet5", "fp32", 16),
    ("vgg16_32", "int8", 8),
    ("vgg16_32", "fp16", 4),
    ("alexnet", "int8", 3),
    ("alexnet", "int16", 1),
    # Net::run_moe through qnb_moe_plan: trunk, gating, 16 expert nets, tail (configs[2])
    ("alexnet_moe", "int8", 3),
])
def test_executor_matches_reference_net(graph, precision, batch):
    r = run(graph, precision, batch)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
