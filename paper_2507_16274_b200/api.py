"""Reference-compatible Python API over libstw (the drop-in boundary).

Names, argument meanings and error behaviour follow the reference package
(`memplan/__init__.py:42-47`, `planner.py:357-505`, `reuse.py:83-93`,
`sim.py:143-238`, `baseline.py:98-137`, `model.py:261-281`). Every compute
call goes through the C-ABI of libstw.so; Python only tensorises inputs and
materialises the reference's value objects from the returned columns.
"""

from __future__ import annotations

import ctypes as C

import os as _os

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


def scan_i64(inp, out=None, inclusive: bool = True, stream=None):
    """Device-wide prefix sum of an int64 device tensor (stw_scan_i64)."""
    out = inp if out is None else out
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_scan_i64(_lib.ptr(inp), _lib.ptr(out), C.c_int64(int(inp.numel())),
                                        C.c_int32(int(inclusive)), _lib.stream_handle(stream), err, C.sizeof(err)),
               err)
    return out


def validate_sets(set_off, t_s, t_e, size, addr, shift: int = 9, stream=None):
    """len(validate_plan(plan)) for every (set, candidate) plan of a batch, on the
    device (K7 over many plans; planner.py:476-505). Device tensors: set_off
    int64 [S+1], t_s/t_e int32 [n] and size int64 [n] in each set's sweep
    order, addr int64 [n_cand, n]. Returns an int64 device tensor [S * n_cand]."""
    import torch

    n_sets = int(set_off.numel()) - 1
    n_cand = int(addr.shape[0]) if addr.dim() == 2 else 1
    count = torch.empty(max(n_sets * n_cand, 1), dtype=torch.int64, device=addr.device)
    rs = _lib.RectSets(n_sets, n_cand, int(t_s.numel()), _lib.ptr(set_off), _lib.ptr(t_s), _lib.ptr(t_e),
                       _lib.ptr(size), _lib.ptr(addr))
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_validate_sets(C.byref(rs), C.c_int32(shift), _lib.ptr(count),
                                             _lib.stream_handle(stream), err, C.sizeof(err)), err)
    return count[: n_sets * n_cand]


# ---------------------------------------------------------------------------
# planner (planner.py:357-505)

import time as _time
from dataclasses import dataclass as _dataclass

from .domain import DEFAULT_ALIGNMENT, PlanError, TraceError
from .plan_types import DecisionColumns, MemoryLayer, PlanStats, StaticPlan, _Keyed


@_dataclass
class BatchPlan:
    """Raw columnar result of stw_plan_batch for T traces x C candidates."""

    batch: HostBatch
    cands: tuple
    rc: np.ndarray        # [T*C]
    err_ids: np.ndarray   # [T*C, 2]
    stats: np.ndarray     # [T*C, NSTATS]
    addr: np.ndarray      # [C, N]
    layer_of: np.ndarray  # [C, N]
    layer_base: np.ndarray
    layer_size: np.ndarray
    fus_tmp: np.ndarray
    fus_avg: np.ndarray
    order: np.ndarray     # [N] trace-local (t_s, id) order
    best_cand: np.ndarray = None
    best_pool: np.ndarray = None
    addr_best: np.ndarray = None


def _cand_bits(cands) -> np.ndarray:
    return np.asarray([(_lib.STW_CAND_FUSION if f else 0) | (_lib.STW_CAND_GAP if g else 0) for f, g in cands],
                      dtype=np.uint8)


def _host_arrays(spec, pinned_from: int = 8 << 20) -> dict:
    """Uninitialised host arrays for the given (name, shape, dtype) fields: one
    page-locked block when they total at least `pinned_from` bytes (device ->
    host copies then run at full link speed), else plain numpy arrays."""
    sizes = [int(np.prod(shape)) * np.dtype(dt).itemsize for _, shape, dt in spec]
    total = sum((z + 63) // 64 * 64 for z in sizes)
    out = {}
    if total >= pinned_from and not _os.environ.get("STW_PAGEABLE_OUT"):
        import torch

        if torch.cuda.is_available():
            raw = torch.empty(total, dtype=torch.uint8, pin_memory=True).numpy()
            off = 0
            for (name, shape, dt), z in zip(spec, sizes):
                out[name] = raw[off:off + z].view(dt).reshape(shape)
                off += (z + 63) // 64 * 64
            return out
    for name, shape, dt in spec:
        out[name] = np.empty(shape, dt)
    return out


def _plan_buffers(hb, cands, alignment, select_best, detail, stream):
    """Host output buffers + the stw_plan_opts/stw_plan_out structs for one batch."""
    C_ = len(cands)
    T, N = hb.T, hb.N
    U = T * C_
    cb = _cand_bits(cands)
    # every field is written in full by the library; large outputs land in one
    # pinned host block (page-locked copies, torch's host allocator caches it)
    spec = [("rc", (U,), np.int32), ("err_ids", (U, 2), np.int64), ("stats", (U, _lib.NSTATS), np.int64),
            ("addr", (C_, N), np.int64), ("order", (N,), np.int32)]
    if detail:
        spec += [("layer_of", (C_, N), np.int32), ("lbase", (C_, N), np.int64), ("lsize", (C_, N), np.int64),
                 ("ftmp", (C_, N), np.float64), ("favg", (C_, N), np.float64)]
    if select_best:
        spec += [("best", (T,), np.int32), ("bpool", (T,), np.int64), ("abest", (N,), np.int64)]
    a = _host_arrays(spec)
    rc, err_ids, stats, addr, order = a["rc"], a["err_ids"], a["stats"], a["addr"], a["order"]
    layer_of, lbase, lsize, ftmp, favg = (a.get(k) for k in ("layer_of", "lbase", "lsize", "ftmp", "favg"))
    best, bpool, abest = (a.get(k) for k in ("best", "bpool", "abest"))
    opts = _lib.PlanOpts(C_, int(select_best), _lib.ptr(cb), alignment,
                         _lib.stream_handle(stream) if stream is not None else None)
    out = _lib.PlanOut(0, _lib.ptr(rc), _lib.ptr(err_ids), _lib.ptr(stats), _lib.ptr(addr), _lib.ptr(layer_of),
                       _lib.ptr(lbase), _lib.ptr(lsize), _lib.ptr(ftmp), _lib.ptr(favg), _lib.ptr(order),
                       _lib.ptr(best), _lib.ptr(abest), _lib.ptr(bpool))
    bp = BatchPlan(hb, tuple(cands), rc, err_ids, stats, addr, layer_of, lbase, lsize, ftmp, favg, order,
                   best, bpool, abest)
    return bp, opts, out, cb


def plan_batch(batch, cands=((True, True),), alignment: int = DEFAULT_ALIGNMENT, select_best: bool = False,
               detail: bool = True, stream=None) -> BatchPlan:
    """Plan every trace of `batch` (HostBatch or list of TraceArrays) under each
    candidate (fusion, gap_insert) on the device (stw_plan_batch)."""
    hb = batch if isinstance(batch, HostBatch) else HostBatch([_arrays_of(t) for t in batch])
    bp, opts, out, _cb = _plan_buffers(hb, cands, alignment, select_best, detail, stream)
    err = _lib.errbuf()
    b = hb.struct()
    _lib.check(_lib.load().stw_plan_batch(C.byref(b), C.byref(opts), C.byref(out), err, C.sizeof(err)), err)
    return bp


def plan_batches(batches, cands=((True, True),), alignment: int = DEFAULT_ALIGNMENT, select_best: bool = False,
                 detail: bool = True, stream=None) -> list:
    """plan_batch over a sequence of batches in one pipelined device call
    (stw_plan_batches: uploads, planning and downloads of neighbouring batches
    overlap). Returns one BatchPlan per batch."""
    hbs = [b if isinstance(b, HostBatch) else HostBatch([_arrays_of(t) for t in b]) for b in batches]
    if not hbs:
        return []
    parts = [_plan_buffers(hb, cands, alignment, select_best, detail, stream) for hb in hbs]
    k = len(hbs)
    bs = (_lib.Batch * k)(*[hb.struct() for hb in hbs])
    outs = (_lib.PlanOut * k)(*[p[2] for p in parts])
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_plan_batches(k, bs, C.byref(parts[0][1]), outs, err, C.sizeof(err)), err)
    return [p[0] for p in parts]


def _unknown_phase_message(ta) -> str:
    """The reference's TraceError text: an event outside [0, horizon]
    (model.py:240-241; checked up front so no kernel indexes past its trace's
    timeline) or the unknown phase (planner.py:390-392 sort order)."""
    out = np.nonzero((ta.t_s < 0) | (ta.t_s >= ta.horizon) | (ta.t_e > ta.horizon))[0]
    if out.size:
        return f"event {int(ta.id[out[0]])}: timestamps outside [0, horizon]"
    n = ta.n_sched
    scoped = np.nonzero((ta.dyn == 0) & (ta.t_e < ta.horizon))[0]
    keys = sorted({(ta.phases[ta.ps[i]], ta.phases[ta.pe[i]]) for i in scoped.tolist()})
    known = set(ta.phases[:n])
    for a, b in keys:
        for ph in (a, b):
            if ph not in known:
                return f"phase {ph} not in schedule"
    return "phase not in schedule"


def raise_unit_error(bp: BatchPlan, t: int, c: int) -> None:
    u = t * len(bp.cands) + c
    rc = int(bp.rc[u])
    if rc == _lib.STW_OK:
        return
    ta = bp.batch.traces[t]
    base = int(bp.batch.ev_off[t])
    e0, e1 = (int(x) for x in bp.err_ids[u])
    if rc == _lib.STW_ETRACE:
        raise TraceError(_unknown_phase_message(ta))
    if e0 >= 0 and e1 < 0:
        i = e0 - base
        raise PlanError(f"event {int(ta.id[i])}: size {int(ta.size[i])} not aligned")
    if e0 >= 0:
        raise PlanError(f"planner emitted conflicting decisions {int(ta.id[e0 - base])} and {int(ta.id[e1 - base])}")
    raise PlanError("pool below the static peak; planner invariant broken")


def _unit_plan(bp: BatchPlan, t: int, c: int, trace, alignment: int, stats) -> StaticPlan:
    raise_unit_error(bp, t, c)
    ta = bp.batch.traces[t]
    u = t * len(bp.cands) + c
    s0, s1 = int(bp.batch.ev_off[t]), int(bp.batch.ev_off[t + 1])
    st = bp.stats[u]
    order = bp.order[s0:s1]
    static = order[ta.dyn[order] == 0]
    addr = bp.addr[c, s0:s1]
    cols = DecisionColumns(ta.id[static], addr[static], ta.size[static], ta.t_s[static], ta.t_e[static], src=static)
    if stats is not None:
        keys = ("num_events", "num_persistent", "num_groups", "num_plans", "num_residuals", "fusion_attempts",
                "fusion_accepted", "gap_insertions", "num_layers", "pool_size", "static_peak")
        for k, v in zip(keys, st[:11].tolist()):
            setattr(stats, k, v)
        na = int(st[6])
        if bp.fus_tmp is not None and na:
            stats.accepted_fusions.extend(zip(bp.fus_tmp[c, s0:s0 + na].tolist(), bp.fus_avg[c, s0:s0 + na].tolist()))
    nl = int(st[8])
    lb = bp.layer_base[c, s0:s0 + nl].copy() if bp.layer_base is not None else np.zeros(nl, np.int64)
    lsz = bp.layer_size[c, s0:s0 + nl].copy() if bp.layer_size is not None else np.zeros(nl, np.int64)
    lay = bp.layer_of[c, s0:s1].copy() if bp.layer_of is not None else None
    events_fn = (lambda tr=trace: tr.events) if trace is not None else ta.to_events

    def layers():
        out = []
        for l in range(nl):
            members = np.nonzero(lay == l)[0] if lay is not None else np.zeros(0, np.int64)

            def slots(members=members):
                ev = events_fn()
                rows = sorted((int(ta.t_s[i]), int(ta.t_e[i]), i) for i in members.tolist())
                return [(a, b, _Keyed(ev[i])) for a, b, i in rows]

            end = int(ta.t_e[members].max()) if members.size else -1
            out.append((int(lb[l]), MemoryLayer(int(lsz[l]), end=end, base=int(lb[l]), slots_fn=slots)))
        return tuple(out)

    return StaticPlan.from_columns(int(st[9]), alignment, cols, events_fn, int(st[11]), layers)


def synthesize_static_plan(trace, *, fusion: bool = True, gap_insert: bool = True,
                           alignment: int = DEFAULT_ALIGNMENT, stats: PlanStats = None) -> StaticPlan:
    """Plan every static request of the trace into a minimal pool (planner.py:357-473)."""
    t0 = _time.monotonic()
    ta = _arrays_of(trace)
    bp = plan_batch([ta], ((fusion, gap_insert),), alignment=alignment)
    if stats is None:
        stats = PlanStats()
    plan = _unit_plan(bp, 0, 0, trace if hasattr(trace, "phase_schedule") else None, alignment, stats)
    stats.plan_seconds = _time.monotonic() - t0
    return plan


def validate_columns(id, addr, size, t_s, t_e) -> np.ndarray:
    """K7 on one plan given as columns (any order): the reference sweep's report
    (planner.py:476-505) as an int array [k, 2] of row indices, in its order."""
    n = int(np.shape(id)[0])
    if n == 0:
        return np.zeros((0, 2), np.int64)
    id = np.ascontiguousarray(id, np.int64)
    addr = np.ascontiguousarray(addr, np.int64)
    size = np.ascontiguousarray(size, np.int64)
    t_s = np.ascontiguousarray(t_s, np.int32)
    t_e = np.ascontiguousarray(t_e, np.int32)
    npairs = C.c_int64(0)
    cap = max(16, 4 * n)
    err = _lib.errbuf()
    L = _lib.load()
    while True:
        pairs = np.empty(2 * cap, np.int32)
        _lib.check(L.stw_validate(C.c_int64(n), _lib.ptr(id), _lib.ptr(addr), _lib.ptr(size), _lib.ptr(t_s),
                                  _lib.ptr(t_e), C.byref(npairs), _lib.ptr(pairs), C.c_int64(cap), None, err,
                                  C.sizeof(err)), err)
        if npairs.value <= cap:
            return pairs[: 2 * npairs.value].reshape(-1, 2).astype(np.int64)
        cap = npairs.value


def validate_plan(plan) -> list:
    """Decision pairs the reference sweep reports as conflicting (planner.py:476-505)."""
    if isinstance(plan, StaticPlan):
        cols = plan.columns()
        decs = plan.decisions
    else:
        decs = tuple(plan.decisions)
        cols = DecisionColumns.from_decisions(decs)
    p = validate_columns(cols.id, cols.addr, cols.size, cols.t_s, cols.t_e).tolist()
    return [(decs[a], decs[b]) for a, b in p]


def peak_live_columns(size, t_s, t_e) -> int:
    """K1 over bare (size, t_s, t_e) columns: max over time of the live bytes
    (model.py:261-276)."""
    n = int(np.shape(size)[0])
    if n == 0:
        return 0
    t_s = np.asarray(t_s, np.int32)
    t_e = np.asarray(t_e, np.int32)
    hz = int(max(int(t_e.max()), int(t_s.max()) + 1, 1))
    z = np.zeros(n, np.int32)
    ta = TraceArrays(np.arange(n, dtype=np.int64), np.asarray(size, np.int64), t_s, t_e, z, z, np.zeros(n, np.uint8),
                     z, z, [None], np.zeros(1, np.int64), np.asarray([hz], np.int64), [], np.zeros(0, np.int64),
                     np.zeros(0, np.int64))
    return peak_live_bytes(ta)


# ---------------------------------------------------------------------------
# dynamic reusable space (reuse.py:42-93)

from .domain import MemplanError as _MemplanError  # noqa: E402
from .ivset import IntervalSet  # noqa: E402
from .plan_types import ReuseEntry, ReuseMap  # noqa: E402


def group_dynamic(events) -> dict:
    """Exact partition of dynamic events by (l_s, l_e) (reuse.py:42-51)."""
    out: dict = {}
    for ev in events:
        if not ev.dynamic or ev.l_s is None or ev.l_e is None:
            raise TraceError(f"event {ev.id}: dynamic event missing layer")
        out.setdefault((ev.l_s, ev.l_e), []).append(ev)
    return out


def _windows(keys, layer_schedule):
    spans = {}
    for s in layer_schedule:
        spans[s.name] = s  # last span wins, like the dict in reuse.py:66
    t_lo, t_hi = [], []
    for key in keys:
        for name in key:
            if name not in spans:
                raise PlanError(f"unknown layer {name!r} in reuse key")
        a, b = spans[key[0]].start, spans[key[1]].end
        if b < a:
            raise PlanError(f"reuse key {key}: free layer ends before alloc layer starts")
        t_lo.append(a)
        t_hi.append(b)
    return np.asarray(t_lo, np.int64), np.asarray(t_hi, np.int64)


def _plan_columns(plan):
    return plan.columns() if isinstance(plan, StaticPlan) else DecisionColumns.from_decisions(tuple(plan.decisions))


def reusable_spaces(cols, t_lo, t_hi, with_cols: bool = False):
    """K8 on the device: idle address intervals of the plan per window."""
    K = int(t_lo.shape[0])
    n = len(cols)
    off = np.zeros(K + 1, np.int64)
    cap = max(16, 2 * (n + 1) * max(K, 1) if n * K < 4_000_000 else 4 * n + 4 * K)
    total = C.c_int64(0)
    err = _lib.errbuf()
    L = _lib.load()
    while True:
        lo = np.empty(cap, np.int64)
        hi = np.empty(cap, np.int64)
        rc = L.stw_reuse_map(C.c_int64(n), _lib.ptr(cols.addr), _lib.ptr(cols.size), _lib.ptr(cols.t_s),
                             _lib.ptr(cols.t_e), C.c_int64(K), _lib.ptr(t_lo), _lib.ptr(t_hi), _lib.ptr(off),
                             _lib.ptr(lo), _lib.ptr(hi), C.c_int64(cap), C.byref(total), None, err, C.sizeof(err))
        if rc == _lib.STW_EARG and total.value > cap:
            cap = total.value
            continue
        _lib.check(rc, err)
        break
    spaces = [IntervalSet.from_bounds(lo[off[k]:off[k + 1]], hi[off[k]:off[k + 1]]) for k in range(K)]
    return spaces if not with_cols else (spaces, (off, lo[:off[K]].copy(), hi[:off[K]].copy()))


def compute_reusable_space(plan, key, layer_schedule):
    """((t_lo, t_hi), idle addresses of the plan over the key's window) (reuse.py:54-80)."""
    t_lo, t_hi = _windows([key], layer_schedule)
    return (int(t_lo[0]), int(t_hi[0])), reusable_spaces(_plan_columns(plan), t_lo, t_hi)[0]


def derive_reuse_map(plan, trace) -> ReuseMap:
    """One reuse entry per dynamic (l_s, l_e) group, empty spaces kept (reuse.py:83-93)."""
    ta = getattr(trace, "_arrays", None)
    if ta is not None:
        keys, _ = ta.dynamic_keys()
    else:
        keys = sorted(group_dynamic(trace.dynamic_events()))
    if not keys:
        return ReuseMap({})
    t_lo, t_hi = _windows(keys, trace.layer_schedule)
    spaces, cols = reusable_spaces(_plan_columns(plan), t_lo, t_hi, with_cols=True)
    rm = ReuseMap({k: ReuseEntry(int(a), int(b), s) for k, a, b, s in zip(keys, t_lo, t_hi, spaces)})
    object.__setattr__(rm, "_cols", (tuple(keys), *cols))  # the device's columns, for the replay's upload
    return rm


def plan_trace(trace, *, fusion=True, gap_insert=True, stats=None):
    """Plan a trace end to end: static plan plus dynamic reuse map (__init__.py:42-47)."""
    plan = synthesize_static_plan(trace, fusion=fusion, gap_insert=gap_insert, stats=stats)
    return plan, derive_reuse_map(plan, trace)


# ---------------------------------------------------------------------------
# replay (sim.py:143-238) and the caching-allocator baseline (baseline.py:98-137)

import json as _json  # noqa: E402
from collections.abc import Sequence as _Sequence  # noqa: E402
from pathlib import Path as _Path  # noqa: E402

from .plan_types import PlanBundle, SimReport  # noqa: E402

_KINDS = ("init", "reserve", "alloc", "free")
_ROUTES = ("planned", "reuse", "fallback", "mismatch", "online")


class ReplayLog(_Sequence):
    """The replay log as the reference's list of dicts, materialised on access
    from the device's columns (sim.py:164, 186, 209-229, 241-253)."""

    def __init__(self, cols: dict, n: int, keys_by_id):
        self._c = cols
        self._n = n
        self._keys_src = keys_by_id  # dict, or a callable making it on first use
        self._keys_d = None
        self._cache = None

    @property
    def _keys(self) -> dict:
        if self._keys_d is None:
            self._keys_d = self._keys_src() if callable(self._keys_src) else self._keys_src
        return self._keys_d

    def __len__(self) -> int:
        return self._n

    def _rec(self, k: int) -> dict:
        c = self._c
        kind = _KINDS[int(c["kind"][k])]
        if kind == "init":
            return {"kind": "init", "pool_size": int(c["size"][k])}
        if kind == "reserve":
            return {"kind": "reserve", "t": int(c["t"][k]), "bytes": int(c["size"][k])}
        rec = {"kind": kind, "t": int(c["t"][k]), "id": int(c["id"][k]), "size": int(c["size"][k]),
               "space": "pool" if c["space"][k] == 0 else "cache", "addr": int(c["addr"][k])}
        if kind == "alloc":
            rec["route"] = _ROUTES[int(c["route"][k])]
            key = self._keys.get(rec["id"])
            if key is not None:
                rec["key"] = list(key)
        return rec

    def _all(self) -> list:
        if self._cache is None:
            self._cache = [self._rec(k) for k in range(self._n)]
        return self._cache

    def __getitem__(self, i):
        if isinstance(i, slice):
            return self._all()[i]
        return self._all()[i] if self._cache is not None else self._rec(range(self._n)[i])

    def __iter__(self):
        return iter(self._all())

    def __eq__(self, other) -> bool:
        return list(self) == list(other)


_LOG_FIELDS = (("t", np.int64), ("id", np.int64), ("size", np.int64), ("addr", np.int64), ("kind", np.int8),
               ("space", np.int8), ("route", np.int8))


def _log_buffers(n: int):
    cap = 1 + 3 * n
    if n >= (1 << 15):
        # a large log comes back over PCIe at page-locked speed: one pinned block
        # (torch's host allocator caches it between calls) carved into the columns
        import torch

        total = sum(cap * np.dtype(dt).itemsize for _, dt in _LOG_FIELDS)
        raw = torch.empty(total, dtype=torch.uint8, pin_memory=True).numpy()
        cols, off = {}, 0
        for name, dt in _LOG_FIELDS:
            nb = cap * np.dtype(dt).itemsize
            cols[name] = raw[off:off + nb].view(dt)
            off += nb
    else:
        cols = {name: np.empty(cap, dt) for name, dt in _LOG_FIELDS}
    lg = _lib.Log(cap, 0, *(_lib.ptr(cols[k]) for k in ("kind", "t", "id", "size", "addr", "space", "route")))
    return lg, cols


def _report(rep) -> SimReport:
    return SimReport(rep.allocated_peak, rep.reserved_peak, rep.efficiency, rep.fragmentation, rep.pool_size,
                     rep.fallback_count, rep.fallback_bytes_peak, rep.reuse_hits, rep.mismatch_count)


def _dyn_keys_by_id(ta) -> dict:
    d = np.nonzero(ta.dyn)[0]
    names = ta.layer_names
    return {int(ta.id[i]): (names[ta.ls[i]], names[ta.le[i]]) for i in d.tolist()}


def _write_log(log, path) -> None:
    with _Path(path).open("w", encoding="utf-8") as fh:
        for rec in log:
            fh.write(_json.dumps(rec, sort_keys=True, separators=(",", ":")) + "\n")


def simulate(trace, plan, *, reuse: bool = True, log_path=None):
    """Replay the trace against a PlanBundle on the device; returns (SimReport, log)."""
    ta = _arrays_of(trace)
    hb = HostBatch([ta])
    cols = getattr(plan, "_cols", None)
    if cols is None:
        cols = DecisionColumns.from_decisions(tuple(plan.decisions))
    bkeys = list(plan.reuse)
    pos = {k: i for i, k in enumerate(bkeys)}
    names, kidx = ta.dynamic_keys()
    key = np.full(len(ta), -1, np.int32)
    if len(names):
        m = kidx >= 0
        key_of_name = np.asarray([pos.get(nm, -1) for nm in names], np.int32)  # one lookup per key, not per event
        key[m] = key_of_name[kidx[m]]
    rc_ = getattr(plan, "_reuse_cols", None)
    if rc_ is not None and rc_[0] == tuple(bkeys):  # the device's reuse columns, same key order
        sp_off, sp_lo, sp_hi = rc_[1], rc_[2], rc_[3]
    else:
        off = [0]
        lo, hi = [], []
        for k in bkeys:
            sp = plan.reuse[k]
            if hasattr(sp, "bounds"):
                a, b = sp.bounds()
                lo.extend(a.tolist())
                hi.extend(b.tolist())
            else:
                for iv in sp:
                    lo.append(iv.lo)
                    hi.append(iv.hi)
            off.append(len(lo))
        sp_off = np.asarray(off, np.int64)
        sp_lo = np.asarray(lo, np.int64)
        sp_hi = np.asarray(hi, np.int64)
    bun = _lib.Bundle(int(plan.pool_size), int(plan.alignment), len(cols), _lib.ptr(cols.id), _lib.ptr(cols.addr),
                      _lib.ptr(cols.size), _lib.ptr(cols.t_s), _lib.ptr(cols.t_e), len(bkeys), _lib.ptr(sp_off),
                      _lib.ptr(sp_lo), _lib.ptr(sp_hi), _lib.ptr(key), int(bool(reuse)))
    rep = _lib.Report()
    lg, lcols = _log_buffers(len(ta))
    eid = C.c_int64(0)
    err = _lib.errbuf()
    b = hb.struct()
    rc = _lib.load().stw_simulate(C.byref(b), C.byref(bun), C.byref(rep), C.byref(lg), C.byref(eid), None, err,
                                  C.sizeof(err))
    if rc == _lib.STW_EPLAN and err.value.startswith(b"reuse entry"):
        k = bkeys[eid.value]
        raise PlanError(f"reuse entry {k} outside pool")
    _lib.check(rc, err)
    log = ReplayLog(lcols, int(lg.len), lambda: _dyn_keys_by_id(ta))
    if log_path is not None:
        _write_log(log, log_path)
    return _report(rep), log


def run_baseline(trace) -> SimReport:
    """Replay every event online through the caching allocator (baseline.py:98-137)."""
    ta = _arrays_of(trace)
    hb = HostBatch([ta])
    rep = _lib.Report()
    eid = C.c_int64(0)
    err = _lib.errbuf()
    b = hb.struct()
    _lib.check(_lib.load().stw_baseline(C.byref(b), C.byref(rep), None, C.byref(eid), None, err, C.sizeof(err)), err)
    return _report(rep)
