"""CPU checks of the drop-in boundary (no GPU needed).

* libqnb.so loads and exports every function include/qnb.h declares.
* The host half of the hot path (requant program, bias conversion inputs, grid
  estimation) is bit-identical to the reference's own functions.
* Without an sm_100 device every compute entry point fails loudly (QNB_E_CUDA) —
  there is no CPU fallback.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2209_15427_b200 import _lib, ops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "qnb.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qnb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert set(names) <= set(_lib.exported_symbols()), set(names) - set(_lib.exported_symbols())


def test_abi_version():
    assert _lib.lib().qnb_abi_version() == 2


def test_host_math_matches_reference(oracle_impl):
    rng = np.random.default_rng(0)
    for trial in range(500):
        dt = _lib.INT8Q if trial % 2 else _lib.INT16Q
        lo = rng.uniform(-1e3, 1e3)
        hi = lo + rng.uniform(1e-3, 1e3)
        a = ops.estimate_params(lo, hi, dt)
        b = oracle_impl.estimate_params(lo, hi, dt)
        assert a.as_tuple() == b.as_tuple()
        c = ops.estimate_from_observation(lo, lo, dt)
        assert c.as_tuple() == oracle_impl.estimate_from_observation(lo, lo, dt).as_tuple()
        q2 = ops.estimate_params(lo - 1, hi + 3, dt)
        q3 = ops.estimate_params(-abs(lo) - 0.5, abs(hi) + 1, dt)
        sb = int(rng.integers(1, 32))
        r = ops.scale_quant_vals(a, q2, q3, sb)
        from oracle.ffi import QVals
        rr = oracle_impl.scale_quant_vals(QVals(*a.as_tuple()), QVals(*q2.as_tuple()), QVals(*q3.as_tuple()), sb)
        assert r.as_tuple() == rr.as_tuple()
        u = ops.scale_quant_vals(a, q3, sb)
        assert u.as_tuple() == oracle_impl.scale_quant_vals(QVals(*a.as_tuple()), QVals(*q3.as_tuple()),
                                                            sb).as_tuple()
        for acc in rng.integers(-(1 << 45), 1 << 45, 8):
            assert ops.requant_clamp(int(acc), r) == oracle_impl.requant_clamp(int(acc), rr)
    for x in (0.5, 1.5, 2.5, -0.5, -1.5, 3.2, 3.7, 1e300, -2.5):
        assert ops.round_half_even(x) == oracle_impl.round_half_even(x)


def test_error_messages_match_reference():
    with pytest.raises(_lib.QnbError, match="shift_bits out of range"):
        ops.scale_quant_vals(ops.estimate_params(0, 1, _lib.INT8Q), ops.estimate_params(0, 1, _lib.INT8Q), 0)
    with pytest.raises(_lib.QnbError, match="degenerate range"):
        ops.estimate_params(1.0, 1.0, _lib.INT8Q)


def _have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu():
    qv = ops.estimate_params(-1, 1, _lib.INT8Q)
    with pytest.raises(_lib.QnbError) as e:
        ops.quantize(np.zeros(8, np.float32), qv, _lib.INT8Q)
    assert e.value.status == 8  # QNB_E_CUDA


def test_net_forward_input_dtype_checks():
    """Net.forward mirrors take_input + the INPUT layer (src/net.cpp:288-302, 394-405):
    a wrong shape is "shape mismatch", a non-float array for a float input is
    "dtype mismatch at blob <top>" (checked before any device work)."""
    from paper_2209_15427_b200 import graphs
    from paper_2209_15427_b200.net import Net
    net = Net(graphs.lenet5(1))
    with pytest.raises(_lib.QnbError, match="shape mismatch"):
        net.forward({"data": np.zeros((2, 1, 27, 28), np.float32)})
    with pytest.raises(_lib.QnbError, match="dtype mismatch at blob data"):
        net.forward({"data": np.zeros((2, 1, 28, 28), np.uint8)})
    inl = next(l for l in net.graph["layers"] if l["kind"] == "input")
    x = np.linspace(-3, 3, 2 * 28 * 28).reshape(2, 1, 28, 28)
    assert Net._input_dtype(x, inl).dtype == np.float32
    assert np.array_equal(Net._input_dtype(x, inl), x.astype(np.float32))
