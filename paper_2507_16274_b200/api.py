"""Reference-compatible Python API over libstw (the drop-in boundary).

Names, argument meanings and error behaviour follow the reference package
(`memplan/__init__.py:42-47`, `planner.py:357-505`, `reuse.py:83-93`,
`sim.py:143-238`, `baseline.py:98-137`, `model.py:261-281`). Every compute
call goes through the C-ABI of libstw.so; Python only tensorises inputs and
materialises the reference's value objects from the returned columns.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .batching import HostBatch
from .soa import TraceArrays, from_events, from_trace


def _arrays_of(obj) -> TraceArrays:
    if isinstance(obj, TraceArrays):
        return obj
    if hasattr(obj, "phase_schedule"):
        return from_trace(obj)
    return from_events(list(obj))


def peak_live_bytes(events) -> int:
    """Max over time of the live bytes (model.py:261-276), computed by K1."""
    ta = _arrays_of(events)
    hb = HostBatch([ta])
    out = np.zeros(1, dtype=np.int64)
    err = _lib.errbuf()
    L = _lib.load()
    b = hb.struct()
    _lib.check(L.stw_peak_live(C.byref(b), C.c_int32(0), _lib.ptr(out), None, err, C.sizeof(err)), err)
    return int(out[0])


def clique_lower_bound(trace) -> int:
    """Peak allocated bytes of the trace; no plan can reserve less (model.py:279-281)."""
    return peak_live_bytes(trace)


def radix_sort_pairs(keys, vals, begin_bit: int = 0, end_bit: int = 64, stream=None) -> None:
    """In-place stable sort of device tensors (uint64 keys as int64, int32 vals) by K2."""
    err = _lib.errbuf()
    L = _lib.load()
    n = int(keys.numel())
    s = _lib.stream_handle(stream)
    _lib.check(L.stw_radix_sort_pairs(_lib.ptr(keys), _lib.ptr(vals), C.c_int64(n), C.c_int32(begin_bit),
                                      C.c_int32(end_bit), s, err, C.sizeof(err)), err)
