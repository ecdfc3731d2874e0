"""B200-native (sm_100a) backend for the QNet mixed-precision inference hot path
(arxiv 2209.15427).  The compute lives in libqnb.so (include/qnb.h); this package
holds its ctypes binding, the host mirror of the reference operator API (ops.py),
the graph/plan compiler (plan.py) and the model fixtures (graphs.py)."""

from ._lib import FP16, FP32, INT8Q, INT16Q, QnbError  # noqa: F401
