"""The reference baseline module's API (`memplan/baseline.py`): the online
caching allocator and `run_baseline`.

`CachingAllocator` is the native allocator core of libstw_alloc.so (the same
C++ policy object the runtime allocator uses for its fallback region,
include/stw_alloc.h `stw_cache_*`); `run_baseline` replays a whole trace
through it on the device (libstw `stw_baseline`, K10).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .api import run_baseline
from .domain import SimulationError

MIN_SEGMENT = 2 * 1024 * 1024  # baseline.py:17

__all__ = ["MIN_SEGMENT", "CachingAllocator", "Segment", "run_baseline"]


@dataclass
class Segment:
    """Snapshot of one reserved segment: base, size and its free blocks (baseline.py:24-32)."""

    base: int
    size: int
    free: list = field(default_factory=list)

    @property
    def end(self) -> int:
        return self.base + self.size


class CachingAllocator:
    """Best-fit/split/merge allocator over lazily reserved power-of-two segments
    (baseline.py:35-95), backed by the native allocator core."""

    def __init__(self, *, base: int = 0, min_segment: int = MIN_SEGMENT) -> None:
        from .runtime import load

        self._L = load()
        self._h = C.c_void_p(self._L.stw_cache_new(int(base), int(min_segment)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._L.stw_cache_delete(h)
            self._h = None

    def _stats(self) -> np.ndarray:
        out = np.zeros(5, np.int64)
        self._L.stw_cache_stats(self._h, out.ctypes.data)
        return out

    @property
    def reserved(self) -> int:
        return int(self._stats()[0])

    @property
    def live_bytes(self) -> int:
        return int(self._stats()[1])

    @property
    def segments(self) -> list:
        st = self._stats()
        ns, nb = int(st[2]), int(st[3])
        base = np.zeros(max(ns, 1), np.int64)
        size = np.zeros(max(ns, 1), np.int64)
        off = np.zeros(ns + 1, np.int64)
        lo = np.zeros(max(nb, 1), np.int64)
        hi = np.zeros(max(nb, 1), np.int64)
        self._L.stw_cache_segments(self._h, base.ctypes.data, size.ctypes.data, off.ctypes.data, lo.ctypes.data,
                                   hi.ctypes.data)
        return [Segment(int(base[g]), int(size[g]),
                        list(zip(lo[off[g]:off[g + 1]].tolist(), hi[off[g]:off[g + 1]].tolist())))
                for g in range(ns)]

    def owns(self, rid: int) -> bool:
        return bool(self._L.stw_cache_owns(self._h, int(rid)))

    def malloc(self, rid: int, size: int) -> tuple:
        """Serve a request; returns (address, newly reserved bytes)."""
        addr = C.c_int64(0)
        grown = C.c_int64(0)
        if self._L.stw_cache_malloc(self._h, int(rid), int(size), C.addressof(addr), C.addressof(grown)):
            raise SimulationError(f"request {rid} already live in cache")
        return addr.value, grown.value

    def free(self, rid: int) -> tuple:
        """Release a request; returns (address, size)."""
        addr = C.c_int64(0)
        size = C.c_int64(0)
        if self._L.stw_cache_free(self._h, int(rid), C.addressof(addr), C.addressof(size)):
            raise SimulationError(f"free of unknown id {rid} in cache")
        return addr.value, size.value
