"""Runtime side of the plan: libstw_alloc.so as a PyTorch
CUDAPluggableAllocator, plus the request-matcher hooks (paper §6).

    rt = PlanAllocator(plan_bundle, trace)        # reserve the pool, load queues + reuse spaces
    rt.install()                                  # torch.cuda.memory.change_current_allocator(...)
    with rt.phase(phase_id):                      # static requests of this phase hit planned offsets
        with rt.layer(("L01.moe.F0", "L01.moe.F0")):   # dynamic requests use the key's reusable space
            ...

Routing is the replay's (sim.py:143-232); `PlanAllocator.replay(trace)` drives
it through a trace's op sequence so its address stream can be compared with
`simulate`'s log.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os

import numpy as np

from . import _lib
from .domain import DeviceError, SimulationError
from .plan_types import DecisionColumns, SimReport
from .soa import from_trace

ALLOC_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstw_alloc.so")
ROUTES = ("planned", "reuse", "fallback", "mismatch")
_alib = None


def load() -> C.CDLL:
    global _alib
    if _alib is None:
        if not os.path.exists(ALLOC_PATH):
            from . import build as _b

            _b.build_alloc()
        L = C.CDLL(ALLOC_PATH)
        L.stw_malloc.restype = C.c_void_p
        L.stw_malloc.argtypes = [C.c_size_t, C.c_int, C.c_void_p]
        L.stw_free.restype = None
        L.stw_free.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
        L.stw_alloc_vaddr.restype = C.c_int64
        L.stw_alloc_vaddr.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.stw_set_phase.restype = None
        L.stw_set_layer.restype = None
        L.stw_alloc_shutdown.restype = C.c_int
        L.stw_cache_new.restype = C.c_void_p
        L.stw_cache_new.argtypes = [C.c_int64, C.c_int64]
        L.stw_cache_delete.restype = None
        L.stw_cache_delete.argtypes = [C.c_void_p]
        L.stw_cache_malloc.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        L.stw_cache_free.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.stw_cache_owns.argtypes = [C.c_void_p, C.c_int64]
        L.stw_cache_stats.restype = None
        L.stw_cache_stats.argtypes = [C.c_void_p, C.c_void_p]
        L.stw_cache_segments.restype = None
        L.stw_cache_segments.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        L.stw_reuse_best_fit.restype = C.c_int64
        L.stw_reuse_best_fit.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_int64]
        _alib = L
    return _alib


class PlanAllocator:
    """Serve a PlanBundle from one reserved pool (plus the fallback region)."""

    def __init__(self, bundle, trace, device: int = 0):
        self.ta = from_trace(trace)
        self.bundle = bundle
        L = load()
        st = self.status()
        if st["initialised"] and st["live"] == 0:
            L.stw_alloc_shutdown()  # nothing points into the old range
            st["initialised"] = 0
        if not st["initialised"]:
            rc = L.stw_alloc_init(C.c_int(device), C.c_int64(int(bundle.pool_size)),
                                  C.c_int64(int(bundle.alignment)))
            if rc != 0:
                raise DeviceError(f"stw_alloc_init failed ({rc})")
        elif st["pool_size"] < int(bundle.pool_size):
            raise DeviceError(f"allocator installed with a {st['pool_size']}-byte pool and {st['live']} live blocks; "
                              f"cannot serve a {int(bundle.pool_size)}-byte plan without freeing them")
        cols = getattr(bundle, "_cols", None) or DecisionColumns.from_decisions(tuple(bundle.decisions))
        # decision -> phase of its event (events_by_id, last one wins: sim.py:156-161); unknown/dynamic ids skipped
        idx = {int(i): k for k, i in enumerate(self.ta.id.tolist())}
        keep, phase = [], []
        for k, i in enumerate(cols.id.tolist()):
            e = idx.get(i)
            if e is not None and not self.ta.dyn[e]:
                keep.append(k)
                phase.append(int(self.ta.ps[e]))
        keep = np.asarray(keep, np.int64)
        self.keys = list(bundle.reuse)
        self.key_index = {k: i for i, k in enumerate(self.keys)}
        off, lo, hi = [0], [], []
        for k in self.keys:
            for iv in bundle.reuse[k]:
                lo.append(iv.lo)
                hi.append(iv.hi)
            off.append(len(lo))
        arr = lambda x, t: np.ascontiguousarray(x, dtype=t)  # noqa: E731
        self._keep = (arr(phase, np.int32), arr(cols.size[keep], np.int64), arr(cols.addr[keep], np.int64),
                      arr(cols.t_s[keep], np.int32), arr(cols.id[keep], np.int64), arr(off, np.int64),
                      arr(lo, np.int64), arr(hi, np.int64))
        ph, sz, ad, ts, ids, o, l_, h_ = self._keep
        rc = L.stw_alloc_load_plan(C.c_int64(len(keep)), _lib.ptr(ph), _lib.ptr(sz), _lib.ptr(ad), _lib.ptr(ts),
                                   _lib.ptr(ids), C.c_int64(len(self.keys)), _lib.ptr(o), _lib.ptr(l_), _lib.ptr(h_))
        if rc != 0:
            raise DeviceError(f"stw_alloc_load_plan failed ({rc})")
        self.phase_index = {p: i for i, p in enumerate(self.ta.phases)}

    # request-matcher hooks -------------------------------------------------
    def set_phase(self, phase) -> None:
        load().stw_set_phase(C.c_int32(self.phase_index[phase] if not isinstance(phase, int) else phase))

    def set_layer(self, key, dynamic: bool = True) -> None:
        load().stw_set_layer(C.c_int32(self.key_index.get(key, -1) if key is not None else -1), C.c_int32(int(dynamic)))

    @contextlib.contextmanager
    def phase(self, phase):
        self.set_phase(phase)
        yield

    @contextlib.contextmanager
    def layer(self, key):
        self.set_layer(key, True)
        try:
            yield
        finally:
            self.set_layer(None, False)

    # torch integration -----------------------------------------------------
    @staticmethod
    def install():
        """Make libstw_alloc the process's CUDA allocator (before any CUDA allocation)."""
        import torch

        alloc = torch.cuda.memory.CUDAPluggableAllocator(ALLOC_PATH, "stw_malloc", "stw_free")
        torch.cuda.memory.change_current_allocator(alloc)
        return alloc

    # introspection ---------------------------------------------------------
    @staticmethod
    def vaddr(ptr: int):
        r = C.c_int32(-1)
        v = load().stw_alloc_vaddr(C.c_void_p(ptr), C.byref(r))
        return int(v), (ROUTES[r.value] if v >= 0 else None)

    @staticmethod
    def report() -> SimReport:
        rep = _lib.Report()
        rc = load().stw_alloc_report(C.byref(rep))
        out = SimReport(rep.allocated_peak, rep.reserved_peak, rep.efficiency, rep.fragmentation, rep.pool_size,
                        rep.fallback_count, rep.fallback_bytes_peak, rep.reuse_hits, rep.mismatch_count)
        if rc == _lib.STW_ESIM:
            st = PlanAllocator.status()
            if st["bad_frees"]:
                raise SimulationError(f"{st['bad_frees']} free(s) of unknown or already freed blocks")
            raise SimulationError("a planned address was occupied at runtime")
        return out

    # replay driver ---------------------------------------------------------
    def replay(self):
        """Issue the trace's allocs/frees in replay order (t, is_alloc, id) through
        stw_malloc/stw_free with the matcher hooks set per request; returns
        [(id, route, vaddr)] of the allocations."""
        ta = self.ta
        L = load()
        n = len(ta)
        t = np.concatenate([ta.t_s, ta.t_e]).astype(np.int64)
        is_alloc = np.concatenate([np.ones(n, np.int64), np.zeros(n, np.int64)])
        ids = np.concatenate([ta.id, ta.id])
        ev = np.concatenate([np.arange(n), np.arange(n)])
        order = np.lexsort((ids, is_alloc, t))
        names, kidx = ta.dynamic_keys()
        ptrs = {}
        out = []
        for o in order.tolist():
            e = int(ev[o])
            if is_alloc[o]:
                if ta.dyn[e]:
                    self.set_layer(names[kidx[e]], True)
                else:
                    L.stw_set_layer(C.c_int32(-1), C.c_int32(0))
                    L.stw_set_phase(C.c_int32(int(ta.ps[e])))
                p = L.stw_malloc(C.c_size_t(int(ta.size[e])), 0, None)
                if not p:
                    raise DeviceError("stw_malloc returned NULL")
                ptrs[e] = p
                out.append((int(ta.id[e]),) + self.vaddr(p)[::-1])
            else:
                L.stw_free(C.c_void_p(ptrs.pop(e)), C.c_size_t(int(ta.size[e])), 0, None)
        L.stw_set_layer(C.c_int32(-1), C.c_int32(0))
        return out

    @staticmethod
    def served() -> list:
        """[(route, replay address)] of every request served since the plan was loaded."""
        L = load()
        L.stw_alloc_served.restype = C.c_int64
        n = L.stw_alloc_served(None, None, C.c_int64(0))
        r = np.empty(n, np.int8)
        v = np.empty(n, np.int64)
        L.stw_alloc_served(_lib.ptr(r), _lib.ptr(v), C.c_int64(n))
        return [(ROUTES[a], b) for a, b in zip(r.tolist(), v.tolist())]

    @staticmethod
    def status() -> dict:
        out = np.zeros(7, np.int64)
        load().stw_alloc_status(_lib.ptr(out))
        keys = ("initialised", "pool_size", "live", "occupied", "bad_frees", "mapped_bytes", "base")
        return {k: int(v) for k, v in zip(keys, out)}

    @staticmethod
    def shutdown() -> None:
        """Release the reserved range; refused while blocks are live."""
        if load().stw_alloc_shutdown() != 0:
            raise DeviceError("stw_alloc_shutdown refused: blocks are still live")
