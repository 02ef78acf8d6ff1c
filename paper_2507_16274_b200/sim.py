"""The reference replay module's API (`memplan/sim.py`): replay of a trace
against a plan, the pool state, dynamic placement and the metrics fold.

`simulate` is the device replay (libstw `stw_simulate`, K9); `compute_metrics`
folds a log on the device (`stw_metrics`); `dynamic_allocate` places through
the runtime allocator's best fit (libstw_alloc `stw_reuse_best_fit`, the code
that serves dynamic requests in the CUDAPluggableAllocator).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Mapping, Optional

import numpy as np

from . import _lib
from .api import ReplayLog, simulate
from .ivset import Interval, IntervalSet
from .plan_types import PlanBundle, SimReport

__all__ = ["PoolState", "SimReport", "compute_metrics", "dynamic_allocate", "simulate", "PlanBundle"]

_KIND = {"init": 0, "reserve": 1, "alloc": 2, "free": 3}
_ROUTE = {"planned": 0, "reuse": 1, "fallback": 2, "mismatch": 3, "online": 4}


@dataclass
class PoolState:
    """Mutable view of the static pool during replay (sim.py:25-36)."""

    pool_size: int
    free: IntervalSet
    live: dict

    @classmethod
    def fresh(cls, pool_size: int) -> "PoolState":
        free = IntervalSet.span(0, pool_size) if pool_size else IntervalSet.empty()
        return cls(pool_size, free, {})


def _log_columns(log):
    if isinstance(log, ReplayLog):
        c = log._c
        n = len(log)
        return (np.ascontiguousarray(c["kind"][:n]), np.ascontiguousarray(c["size"][:n]),
                np.ascontiguousarray(c["space"][:n]), np.ascontiguousarray(c["route"][:n]))
    recs = list(log)
    n = len(recs)
    kind = np.full(n, -1, np.int8)
    size = np.zeros(n, np.int64)
    space = np.zeros(n, np.int8)
    route = np.full(n, -1, np.int8)
    for i, r in enumerate(recs):
        k = _KIND.get(r["kind"], -1)
        kind[i] = k
        if k == 0:
            size[i] = r["pool_size"]
        elif k == 1:
            size[i] = r["bytes"]
        elif k >= 2:
            size[i] = r["size"]
            space[i] = 1 if r["space"] == "cache" else 0
            if k == 2:
                route[i] = _ROUTE.get(r["route"], -1)
    return kind, size, space, route


def compute_metrics(log: Iterable[dict]) -> SimReport:
    """Fold a replay log into a report (sim.py:67-117), on the device."""
    kind, size, space, route = _log_columns(log)
    rep = _lib.Report()
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_metrics(C.c_int64(len(kind)), _lib.ptr(kind), _lib.ptr(size), _lib.ptr(space),
                                       _lib.ptr(route), C.byref(rep), None, err, C.sizeof(err)), err)
    return SimReport(rep.allocated_peak, rep.reserved_peak, rep.efficiency, rep.fragmentation, rep.pool_size,
                     rep.fallback_count, rep.fallback_bytes_peak, rep.reuse_hits, rep.mismatch_count)


def _bounds(ivs) -> tuple:
    lo = np.ascontiguousarray([iv.lo for iv in ivs], np.int64)
    hi = np.ascontiguousarray([iv.hi for iv in ivs], np.int64)
    return lo, hi


def dynamic_allocate(state: PoolState, reuse_spaces: Mapping, key, size: int) -> Optional[int]:
    """Place a dynamic request at the low end of the best-fit piece of
    free ∩ reuse space, or return None for the fallback path (sim.py:120-140)."""
    space = reuse_spaces.get(key)
    if space is None or not space:
        return None
    from .runtime import load

    flo, fhi = _bounds(state.free)
    slo, shi = _bounds(space)
    lo = load().stw_reuse_best_fit(len(flo), flo.ctypes.data, fhi.ctypes.data, len(slo), slo.ctypes.data,
                                   shi.ctypes.data, int(size))
    if lo < 0:
        return None
    state.free = state.free.remove(Interval(int(lo), int(lo) + size))
    return int(lo)
