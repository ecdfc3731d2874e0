import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; runs the CUDA kernels")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def restatement():
    from oracle import ffi
    return ffi.Restatement()


@pytest.fixture(scope="session")
def reference():
    from oracle import ffi
    if not ffi.have_reference():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return ffi.Reference()


@pytest.fixture(scope="session")
def oracle_impl():
    """The strongest available checker: the compiled reference, else the restatement."""
    from oracle import ffi
    return ffi.Reference() if ffi.have_reference() else ffi.Restatement()


@pytest.fixture(scope="session")
def qnb_ops():
    from paper_2209_15427_b200 import ops
    return ops
