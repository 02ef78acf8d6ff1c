"""The reference file-format module's API (`memplan/traceio.py`): JSONL trace
files (raw / paired layouts) and JSON plan files, read and written by the
native libstw_io.so (include/stw_io.h) straight to / from the columns libstw
consumes -- no per-event objects on the way.

Error behaviour is the reference's (TraceError / PlanError with the same
text). The native reader reports which line failed to decode or convert; the
exact exception text of that one line is then re-derived here with Python's
own json / int() / str() (`_explain_*`), so messages match the reference's
byte for byte.
"""

from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path

import numpy as np

from .domain import DEFAULT_ALIGNMENT, PhaseId, PlanError, Trace, TraceError, align_up
from .ivset import Interval, IntervalSet
from .plan_types import PlanBundle, PlanDecision
from .soa import TraceArrays, from_trace

SCHEMA_VERSION = 1

__all__ = ["SCHEMA_VERSION", "PlanBundle", "PlanDecision", "parse_trace", "read_plan", "write_plan", "write_trace"]

IO_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstw_io.so")
IOE_MSG, IOE_JSON, IOE_RECORD, IOE_HEADER, IOE_OS, IOE_PLANDOC, IOE_INDEX, IOE_TYPE = range(1, 9)


class IoError(C.Structure):
    _fields_ = [("kind", C.c_int32), ("line", C.c_int64), ("text", C.c_char * 1024)]


class TraceCols(C.Structure):
    _fields_ = [("n", C.c_int64)] + [(k, C.c_void_p) for k in ("id", "size", "t_s", "t_e", "ps", "pe", "ls", "le",
                                                              "dyn")] + [
        ("n_tags", C.c_int64), ("tags", C.c_void_p), ("n_sched", C.c_int64), ("ph_start", C.c_void_p),
        ("ph_end", C.c_void_p), ("n_names", C.c_int64), ("names", C.c_void_p), ("n_layers", C.c_int64),
        ("ly_start", C.c_void_p), ("ly_end", C.c_void_p)]


class PlanCols(C.Structure):
    _fields_ = [("pool_size", C.c_int64), ("alignment", C.c_int64), ("n_dec", C.c_int64)] + [
        (k, C.c_void_p) for k in ("id", "addr", "size", "t_s", "t_e")] + [
        ("n_keys", C.c_int64), ("l_s", C.c_void_p), ("l_e", C.c_void_p), ("iv_off", C.c_void_p),
        ("iv_lo", C.c_void_p), ("iv_hi", C.c_void_p)]


_io = None


def load() -> C.CDLL:
    global _io
    if _io is None:
        if not os.path.exists(IO_PATH):
            from . import build as _b

            _b.build_io()
        L = C.CDLL(IO_PATH)
        for name in ("stw_trace_read", "stw_trace_write", "stw_plan_write", "stw_plan_read"):
            getattr(L, name).restype = C.c_int
        L.stw_trace_phase_tag.restype = C.c_char_p
        L.stw_trace_layer_name.restype = C.c_char_p
        L.stw_plan_key.restype = C.c_char_p
        for name in ("stw_trace_free", "stw_trace_sizes", "stw_trace_events", "stw_trace_schedules", "stw_plan_free",
                     "stw_plan_sizes", "stw_plan_decisions", "stw_plan_reuse"):
            getattr(L, name).restype = None
        _io = L
    return _io


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _cstrs(strs):
    enc = [s.encode("utf-8") for s in strs]
    arr = (C.c_char_p * max(len(enc), 1))(*enc)
    return arr, enc


def _os_error(e: IoError, path):
    raise OSError(int(e.line), os.strerror(int(e.line)), str(path))


# ---------------------------------------------------------------------------
# trace files


def _lines(path):
    return Path(path).read_text(encoding="utf-8").splitlines()


def _decode(where: str, line: str, err_cls):
    try:
        return json.loads(line)
    except json.JSONDecodeError as exc:
        raise err_cls(f"{where}: {exc}") from None


def _explain_trace(path: str, e: IoError):
    """Raise the reference's exception for the line the native reader flagged."""
    lines = _lines(path)
    k = int(e.line)
    if e.kind == IOE_JSON:
        json.loads(lines[k - 1])  # re-raised below with the reference's wording
        raise TraceError(f"{path}:{k}: malformed line")  # pragma: no cover (native/json disagree)
    if e.kind == IOE_HEADER:
        header = json.loads(lines[0])
        what = e.text.decode()
        if what == "version":
            raise TraceError(f"{path}: unsupported schema version {header.get('version')}")
        if what == "format":
            raise TraceError(f"{path}: unknown trace format {header.get('format', 'raw')!r}")
        try:
            tuple((PhaseId.parse(tag), int(s), int(t)) for tag, s, t in header["phases"])
            tuple((str(n), int(s), int(t)) for n, s, t in header.get("layers", []))
        except (KeyError, TypeError, ValueError) as exc:
            raise TraceError(f"{path}: malformed paired header: {exc}") from None
        raise TraceError(f"{path}: paired header value not supported by the native reader")
    rec = json.loads(lines[k - 1])
    fmt = json.loads(lines[0]).get("format", "raw")
    if fmt == "raw":
        try:
            op = rec["op"]
            int(rec["id"])
            PhaseId.parse(rec["phase"])
        except (KeyError, TypeError, ValueError) as exc:
            raise TraceError(f"{path}:{k}: malformed record: {exc}") from None
        if op == "alloc":
            try:
                align_up(int(rec["size"]))
            except (KeyError, TypeError, ValueError) as exc:
                raise TraceError(f"{path}:{k}: bad size: {exc}") from None
        elif op != "free":
            raise TraceError(f"{path}:{k}: unknown op {op!r}")
    else:
        try:
            int(rec["id"]), align_up(int(rec["size"])), int(rec["t_s"]), int(rec["t_e"])
            PhaseId.parse(rec["p_s"]), PhaseId.parse(rec["p_e"]), bool(rec["dynamic"])
        except (KeyError, TypeError, ValueError) as exc:
            raise TraceError(f"{path}:{k}: malformed record: {exc}") from None
    raise TraceError(f"{path}:{k}: record value not supported by the native reader")


def _raise_io(e: IoError, path: str, err_cls, explain):
    if e.kind == IOE_OS:
        _os_error(e, path)
    if e.kind == IOE_MSG:
        raise err_cls(e.text.decode("utf-8", errors="replace"))
    if e.kind == IOE_TYPE:
        raise TypeError(e.text.decode("utf-8", errors="replace"))
    if e.kind == IOE_JSON and err_cls is TraceError:
        lines = _lines(path)
        _decode(f"{path}:{int(e.line)}: malformed line", lines[int(e.line) - 1], TraceError)
    explain(path, e)
    raise err_cls(e.text.decode())  # pragma: no cover


def parse_trace(path) -> Trace:
    """Read a trace file (raw or paired layout) into a validated Trace
    (traceio.py:48-68; Trace.validate, model.py:219-251)."""
    p = str(Path(path))
    L = load()
    h = C.c_void_p()
    e = IoError()
    if L.stw_trace_read(p.encode(), C.byref(h), C.byref(e)) != 0:
        _raise_io(e, p, TraceError, _explain_trace)
    try:
        z = np.zeros(5, np.int64)
        L.stw_trace_sizes(h, _p(z))
        n, ntags, nsched, nnames, nknown = (int(x) for x in z)
        i64 = lambda: np.empty(n, np.int64)  # noqa: E731
        i32 = lambda: np.empty(n, np.int32)  # noqa: E731
        id_, size, ts, te = i64(), i64(), i64(), i64()
        ps, pe, ls, le = i32(), i32(), i32(), i32()
        dyn = np.empty(n, np.uint8)
        L.stw_trace_events(h, *(_p(a) for a in (id_, size, ts, te, ps, pe, dyn, ls, le)))
        ph_s, ph_e = np.empty(nsched, np.int64), np.empty(nsched, np.int64)
        ly_s, ly_e = np.empty(nknown, np.int64), np.empty(nknown, np.int64)
        L.stw_trace_schedules(h, _p(ph_s), _p(ph_e), _p(ly_s), _p(ly_e))
        tags = [L.stw_trace_phase_tag(h, k).decode() for k in range(ntags)]
        names = [L.stw_trace_layer_name(h, k).decode() for k in range(nnames)]
    finally:
        L.stw_trace_free(h)
    i32max = np.iinfo(np.int32).max
    if n and (ts.min() < 0 or te.max() > i32max):
        raise TraceError("timestamps outside the supported int32 range")
    ta = TraceArrays(id_, size, ts.astype(np.int32), te.astype(np.int32), ps, pe, dyn, ls, le,
                     [PhaseId.parse(t) for t in tags], ph_s, ph_e, names, ly_s, ly_e, nknown)
    return Trace.from_arrays(ta)


def _trace_cols(trace):
    ta = trace if isinstance(trace, TraceArrays) else from_trace(trace)
    tags, tag_keep = _cstrs([p.tag() for p in ta.phases])
    names, name_keep = _cstrs(ta.layer_names)
    k = len(ta.layer_names) if ta.n_known_layers < 0 else ta.n_known_layers
    arrs = dict(id=np.ascontiguousarray(ta.id, np.int64), size=np.ascontiguousarray(ta.size, np.int64),
                t_s=np.ascontiguousarray(ta.t_s, np.int64), t_e=np.ascontiguousarray(ta.t_e, np.int64),
                ps=np.ascontiguousarray(ta.ps, np.int32), pe=np.ascontiguousarray(ta.pe, np.int32),
                ls=np.ascontiguousarray(ta.ls, np.int32), le=np.ascontiguousarray(ta.le, np.int32),
                dyn=np.ascontiguousarray(ta.dyn, np.uint8),
                ph_s=np.ascontiguousarray(ta.phase_start, np.int64), ph_e=np.ascontiguousarray(ta.phase_end, np.int64),
                ly_s=np.ascontiguousarray(ta.layer_start[:k], np.int64),
                ly_e=np.ascontiguousarray(ta.layer_end[:k], np.int64))
    c = TraceCols(len(ta), *(_p(arrs[x]) for x in ("id", "size", "t_s", "t_e", "ps", "pe", "ls", "le", "dyn")),
                  len(ta.phases), C.cast(tags, C.c_void_p), ta.n_sched, _p(arrs["ph_s"]), _p(arrs["ph_e"]),
                  len(ta.layer_names), C.cast(names, C.c_void_p), k, _p(arrs["ly_s"]), _p(arrs["ly_e"]))
    return c, (arrs, tags, tag_keep, names, name_keep)


def write_trace(trace, path, form: str = "raw") -> None:
    """Serialize a trace (traceio.py:222-291); the raw layout requires every
    timestamp in [0, horizon) to hold exactly one op."""
    if form not in ("raw", "paired"):
        raise ValueError(f"unknown trace format {form!r}")
    c, _keep = _trace_cols(trace)
    e = IoError()
    p = str(Path(path))
    if load().stw_trace_write(C.byref(c), 0 if form == "raw" else 1, p.encode(), C.byref(e)) != 0:
        if e.kind == IOE_INDEX:
            raise IndexError("list index out of range")
        _raise_io(e, p, TraceError, lambda *_: None)


# ---------------------------------------------------------------------------
# plan files


def write_plan(bundle, path) -> None:
    """Canonical plan file (traceio.py:334-354): sort_keys, indent=2."""
    cols = getattr(bundle, "_cols", None)
    if cols is not None:
        dec = [np.ascontiguousarray(getattr(cols, k), np.int64) for k in ("id", "addr", "size", "t_s", "t_e")]
    else:
        ds = tuple(bundle.decisions)
        dec = [np.fromiter((getattr(d, k) for d in ds), np.int64, len(ds)) for k in ("id", "addr", "size", "t_s", "t_e")]
    keys = list(bundle.reuse)
    ls, ls_keep = _cstrs([str(k[0]) for k in keys])
    le, le_keep = _cstrs([str(k[1]) for k in keys])
    off, lo, hi = [0], [], []
    for k in keys:
        for iv in bundle.reuse[k]:
            lo.append(iv.lo)
            hi.append(iv.hi)
        off.append(len(lo))
    off, lo, hi = (np.asarray(x, np.int64) for x in (off, lo, hi))
    pc = PlanCols(int(bundle.pool_size), int(bundle.alignment), len(dec[0]), *(_p(a) for a in dec), len(keys),
                  C.cast(ls, C.c_void_p), C.cast(le, C.c_void_p), _p(off), _p(lo), _p(hi))
    e = IoError()
    p = str(Path(path))
    if load().stw_plan_write(C.byref(pc), p.encode(), C.byref(e)) != 0:
        _raise_io(e, p, PlanError, lambda *_: None)


def _explain_plan(path: str, e: IoError):
    doc = json.loads(Path(path).read_text(encoding="utf-8"))
    if e.kind == IOE_HEADER:
        raise PlanError(f"{path}: unsupported schema version {doc.get('version')}")
    if doc.get("version") != SCHEMA_VERSION:
        raise PlanError(f"{path}: unsupported schema version {doc.get('version')}")
    try:
        decs = tuple(PlanDecision(int(d["id"]), int(d["addr"]), int(d["size"]), int(d["t_s"]), int(d["t_e"]))
                     for d in doc["decisions"])
        {(str(r["l_s"]), str(r["l_e"])): IntervalSet(Interval(int(a), int(b)) for a, b in r["intervals"])
         for r in doc.get("reuse_map", [])}
        bundle = PlanBundle(int(doc["pool_size"]), int(doc.get("alignment", DEFAULT_ALIGNMENT)), decs, {})
    except (KeyError, TypeError, ValueError) as exc:
        raise PlanError(f"{path}: malformed plan file: {exc}") from None
    bundle.validate()
    raise PlanError(f"{path}: plan value not supported by the native reader")


def read_plan(path) -> PlanBundle:
    """Read and validate a plan file (traceio.py:357-391)."""
    p = str(Path(path))
    L = load()
    h = C.c_void_p()
    e = IoError()
    if L.stw_plan_read(p.encode(), C.byref(h), C.byref(e)) != 0:
        if e.kind == IOE_JSON:
            _decode(f"{p}: malformed plan file", Path(p).read_text(encoding="utf-8"), PlanError)
        _raise_io(e, p, PlanError, _explain_plan)
    try:
        z = np.zeros(5, np.int64)
        L.stw_plan_sizes(h, _p(z))
        pool, align, nd, nk, niv = (int(x) for x in z)
        cols = [np.empty(nd, np.int64) for _ in range(5)]
        L.stw_plan_decisions(h, *(_p(a) for a in cols))
        off = np.empty(nk + 1, np.int64)
        lo, hi = np.empty(niv, np.int64), np.empty(niv, np.int64)
        L.stw_plan_reuse(h, _p(off), _p(lo), _p(hi))
        keys = [(L.stw_plan_key(h, k, 0).decode(), L.stw_plan_key(h, k, 1).decode()) for k in range(nk)]
    finally:
        L.stw_plan_free(h)
    from .plan_types import DecisionColumns

    decisions = tuple(PlanDecision(*row) for row in zip(*(c.tolist() for c in cols)))
    reuse = {k: IntervalSet(Interval(a, b) for a, b in zip(lo[off[i]:off[i + 1]].tolist(),
                                                           hi[off[i]:off[i + 1]].tolist()))
             for i, k in enumerate(keys)}
    bundle = PlanBundle(pool, align, decisions, reuse)
    for key, space in reuse.items():
        for iv in space:
            if iv.lo < 0 or iv.hi > pool:
                raise PlanError(f"reuse entry {key} outside pool")
    object.__setattr__(bundle, "_cols", DecisionColumns(*cols))
    return bundle
