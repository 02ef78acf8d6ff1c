"""TEST INFRASTRUCTURE ONLY -- ctypes front-end of the C parity oracle.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module. It wraps liboracle.so (built from stw_oracle.c by oracle/Makefile
or __graft_entry__.build()) and speaks the SoA layout of
paper_2507_16274_b200.soa.TraceArrays.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

OK, TRACE_ERROR, PLAN_ERROR, SIM_ERROR = 0, 1, 2, 3


class OracleTrace(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("id", C.c_void_p), ("size", C.c_void_p),
        ("t_s", C.c_void_p), ("t_e", C.c_void_p), ("ps", C.c_void_p), ("pe", C.c_void_p),
        ("dyn", C.c_void_p),
        ("horizon", C.c_int32), ("n_sched", C.c_int32),
    ]


class OracleStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "num_events", "num_persistent", "num_groups", "num_plans", "num_residuals",
        "fusion_attempts", "fusion_accepted", "gap_insertions", "num_layers",
        "pool_size", "static_peak", "persistent_size", "n_accepted")]


class OracleLog(C.Structure):
    _fields_ = [("cap", C.c_int64), ("len", C.c_int64), ("kind", C.c_void_p), ("t", C.c_void_p),
                ("id", C.c_void_p), ("size", C.c_void_p), ("addr", C.c_void_p),
                ("space", C.c_void_p), ("route", C.c_void_p), ("key", C.c_void_p)]


class OracleReport(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "allocated_peak", "reserved_peak", "pool_size", "fallback_count", "fallback_bytes_peak",
        "reuse_hits", "mismatch_count")] + [("efficiency", C.c_double), ("fragmentation", C.c_double)]


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "stw_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        L.or_peak_live.restype = C.c_int64
        L.or_peak_live.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_plan.restype = C.c_int
        L.or_validate.restype = C.c_int64
        L.or_reuse.restype = C.c_int64
        L.or_simulate.restype = C.c_int
        L.or_baseline.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _trace_struct(ta):
    cols = dict(
        id=_c(ta.id, np.int64), size=_c(ta.size, np.int64), t_s=_c(ta.t_s, np.int32),
        t_e=_c(ta.t_e, np.int32), ps=_c(ta.ps, np.int32), pe=_c(ta.pe, np.int32),
        dyn=_c(ta.dyn, np.uint8),
    )
    s = OracleTrace(len(ta), *(_p(cols[k]) for k in ("id", "size", "t_s", "t_e", "ps", "pe", "dyn")),
                    ta.horizon, ta.n_sched)
    return s, cols


def peak_live(size, t_s, t_e) -> int:
    size, t_s, t_e = _c(size, np.int64), _c(t_s, np.int32), _c(t_e, np.int32)
    return int(lib().or_peak_live(C.c_int64(size.shape[0]), _p(size), _p(t_s), _p(t_e)))


@dataclass
class OraclePlan:
    rc: int
    err: str
    addr: np.ndarray
    layer_of: np.ndarray
    layer_base: np.ndarray
    layer_size: np.ndarray
    stats: dict
    accepted: list = field(default_factory=list)


def plan(ta, fusion=True, gap_insert=True, alignment=512) -> OraclePlan:
    s, keep = _trace_struct(ta)
    n = len(ta)
    addr = np.empty(n, np.int64)
    layer_of = np.empty(n, np.int32)
    cap = max(16, n + 1)
    lb = np.empty(cap, np.int64)
    ls = np.empty(cap, np.int64)
    ft = np.empty(cap, np.float64)
    fa = np.empty(cap, np.float64)
    st = OracleStats()
    err = C.create_string_buffer(512)
    rc = lib().or_plan(C.byref(s), C.c_int(int(fusion)), C.c_int(int(gap_insert)), C.c_int64(alignment),
                       _p(addr), _p(layer_of), _p(lb), _p(ls), C.c_int64(cap), _p(ft), _p(fa),
                       C.c_int64(cap), C.byref(st), err, C.c_size_t(512))
    stats = {k: int(getattr(st, k)) for k, _ in OracleStats._fields_}
    nl = stats["num_layers"]
    na = stats["n_accepted"]
    return OraclePlan(rc, err.value.decode(), addr, layer_of, lb[:nl].copy(), ls[:nl].copy(), stats,
                      list(zip(ft[:na].tolist(), fa[:na].tolist())))


def validate(id, addr, size, t_s, t_e, cap=1 << 20):
    id, addr, size = _c(id, np.int64), _c(addr, np.int64), _c(size, np.int64)
    t_s, t_e = _c(t_s, np.int32), _c(t_e, np.int32)
    pairs = np.empty(2 * cap, np.int32)
    n = lib().or_validate(C.c_int64(id.shape[0]), _p(id), _p(addr), _p(size), _p(t_s), _p(t_e),
                          _p(pairs), C.c_int64(cap))
    return int(n), pairs[: 2 * min(n, cap)].reshape(-1, 2)


def reuse(addr, size, t_s, t_e, t_lo, t_hi):
    addr, size = _c(addr, np.int64), _c(size, np.int64)
    t_s, t_e = _c(t_s, np.int32), _c(t_e, np.int32)
    t_lo, t_hi = _c(t_lo, np.int64), _c(t_hi, np.int64)
    K = t_lo.shape[0]
    cap = 4 * (addr.shape[0] + 2) * max(K, 1)
    off = np.empty(K + 1, np.int64)
    lo = np.empty(cap, np.int64)
    hi = np.empty(cap, np.int64)
    tot = lib().or_reuse(C.c_int64(addr.shape[0]), _p(addr), _p(size), _p(t_s), _p(t_e), C.c_int64(K),
                         _p(t_lo), _p(t_hi), _p(off), _p(lo), _p(hi), C.c_int64(cap))
    assert tot >= 0
    return off, lo[:tot].copy(), hi[:tot].copy()


@dataclass
class OracleReplay:
    rc: int
    err: str
    err_id: int
    report: dict
    log: dict


def _mk_log(cap):
    cols = dict(kind=np.empty(cap, np.int8), t=np.empty(cap, np.int64), id=np.empty(cap, np.int64),
                size=np.empty(cap, np.int64), addr=np.empty(cap, np.int64), space=np.empty(cap, np.int8),
                route=np.empty(cap, np.int8), key=np.empty(cap, np.int32))
    lg = OracleLog(cap, 0, *(_p(cols[k]) for k in ("kind", "t", "id", "size", "addr", "space", "route", "key")))
    return lg, cols


def _finish(rc, err, eid, rep, lg, cols):
    n = min(lg.len, lg.cap)
    report = {k: getattr(rep, k) for k, _ in OracleReport._fields_}
    return OracleReplay(rc, err.value.decode(), int(eid.value), report, {k: v[:n].copy() for k, v in cols.items()})


def simulate(ta, key, pool_size, alignment, d_id, d_addr, d_size, d_ts, d_te, sp_off, sp_lo, sp_hi, reuse=True):
    s, keep = _trace_struct(ta)
    key = _c(key, np.int32)
    d_id, d_addr, d_size = _c(d_id, np.int64), _c(d_addr, np.int64), _c(d_size, np.int64)
    d_ts, d_te = _c(d_ts, np.int32), _c(d_te, np.int32)
    sp_off, sp_lo, sp_hi = _c(sp_off, np.int64), _c(sp_lo, np.int64), _c(sp_hi, np.int64)
    cap = 3 * len(ta) + 8
    lg, cols = _mk_log(cap)
    rep = OracleReport()
    eid = C.c_int64(0)
    err = C.create_string_buffer(512)
    rc = lib().or_simulate(C.byref(s), _p(key), C.c_int64(pool_size), C.c_int64(alignment),
                           C.c_int64(d_id.shape[0]), _p(d_id), _p(d_addr), _p(d_size), _p(d_ts), _p(d_te),
                           C.c_int64(sp_off.shape[0] - 1), _p(sp_off), _p(sp_lo), _p(sp_hi), C.c_int(int(reuse)),
                           C.byref(rep), C.byref(lg), C.byref(eid), err, C.c_size_t(512))
    return _finish(rc, err, eid, rep, lg, cols)


def baseline(ta):
    s, keep = _trace_struct(ta)
    cap = 3 * len(ta) + 8
    lg, cols = _mk_log(cap)
    rep = OracleReport()
    eid = C.c_int64(0)
    err = C.create_string_buffer(512)
    rc = lib().or_baseline(C.byref(s), C.byref(rep), C.byref(lg), C.byref(eid), err, C.c_size_t(512))
    return _finish(rc, err, eid, rep, lg, cols)
