"""QCNM model store (include/qnet/model_store.hpp:29-60, src/model_store.cpp) over the
C-ABI reader/writer in libqnb (qnb_model_*).  load_model maps the file: every
record's payload is a numpy view into the mapping, so a plan compiled from a loaded
Net packs the weights from the file bytes straight into device tiles.

    m = load_model("alexnet_int8.qcnm")
    net.load_weights(m)            # Net::load_weights, src/net.cpp:605-619
    save_model(net.to_model(), p)  # Net::to_model + save_model, src/net.cpp:546-603
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import QVals, check

NP_OF = {0: np.float32, 1: np.uint16, 2: np.uint8, 3: np.uint16}
WIDTH = {0: 4, 1: 2, 2: 1, 3: 2}
I_RANGE = {0: (0, 0), 1: (0, 0), 2: (0, 255), 3: (0, 65535)}


@dataclass
class ParamRecord:
    """qnet::ParamRecord (include/qnet/model_store.hpp:33-43)."""

    name: str
    dtype: int = 0
    extents: tuple = ()
    f_min: float = 0.0
    f_max: float = 0.0
    scale: float = 0.0
    zero: float = 0.0
    one: float = 0.0
    payload: np.ndarray = field(default_factory=lambda: np.empty(0, np.uint8))

    def array(self) -> np.ndarray:
        """The payload as a tensor of the record's dtype and extents (a view)."""
        return self.payload.view(NP_OF[self.dtype]).reshape(self.extents)


def _f32(x: float) -> float:
    return float(np.float32(x))


def set_record_qvals(rec: ParamRecord, qv) -> None:
    """src/model_store.cpp:106-112 (fields narrowed to float)."""
    rec.f_min, rec.f_max, rec.scale = _f32(qv.f_min), _f32(qv.f_max), _f32(qv.scale)
    rec.zero, rec.one = _f32(qv.zero), _f32(qv.one)


def record_qvals(rec: ParamRecord) -> QVals:
    """src/model_store.cpp:114-124: zero = lround(zero), integer range of the dtype."""
    z = rec.zero
    zi = int(math.copysign(math.floor(abs(z) + 0.5), z))
    lo, hi = I_RANGE[rec.dtype]
    return QVals(rec.f_min, rec.f_max, rec.scale, zi, rec.one, lo, hi)


class _Mapping:
    """Owns one qnb_model handle (the file mapping); unmapped when the last Model or
    payload view referencing it is gone."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        try:
            if self.h:
                L.lib().qnb_model_close(self.h)
        except Exception:
            pass


class Model:
    """qnet::Model.  A loaded model's payloads are views into the file mapping; every
    view holds a reference to the mapping, so it stays valid after the Model is gone."""

    def __init__(self, records=None, _mapping=None):
        self.records = list(records or [])
        self._mapping = _mapping

    def find(self, name: str):
        return next((r for r in self.records if r.name == name), None)


def load_model(path: str) -> Model:
    lib = L.lib()
    h = C.c_void_p()
    check(lib.qnb_model_open(str(path).encode(), C.byref(h)))
    mapping = _Mapping(h)
    n = C.c_int64()
    check(lib.qnb_model_count(h, C.byref(n)))
    recs = []
    for i in range(n.value):
        r = L.Record()
        check(lib.qnb_model_record(h, i, C.byref(r)))
        if r.payload_bytes:
            buf = (C.c_uint8 * r.payload_bytes).from_address(r.payload)
            buf._mapping = mapping  # the view's base chain keeps the mapping alive
            payload = np.frombuffer(buf, np.uint8)
            payload.flags.writeable = False  # the mapping is read-only
        else:
            payload = np.empty(0, np.uint8)
        recs.append(ParamRecord(r.name.decode(), r.dtype, tuple(r.extents[: r.rank]), r.f_min, r.f_max,
                                r.scale, r.zero, r.one, payload))
    return Model(recs, mapping)


def save_model(m: Model, path: str) -> None:
    arr = (L.Record * max(len(m.records), 1))()
    keep = []
    for i, r in enumerate(m.records):
        e = arr[i]
        nb = r.name.encode()
        keep.append(nb)
        e.name = nb
        e.dtype, e.rank = r.dtype, len(r.extents)
        for d, x in enumerate(r.extents):
            e.extents[d] = int(x)
        e.f_min, e.f_max, e.scale, e.zero, e.one = r.f_min, r.f_max, r.scale, r.zero, r.one
        p = np.ascontiguousarray(r.payload).view(np.uint8).reshape(-1)
        keep.append(p)
        e.payload = p.ctypes.data if p.size else None
        e.payload_bytes = p.size
    check(L.lib().qnb_model_save(str(path).encode(), arr, len(m.records)))
