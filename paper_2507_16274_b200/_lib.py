"""ctypes binding of libstw.so (include/stw.h).

The shared library is built in-tree (build.py) and is the only compute path:
if it is missing or no CUDA device is usable, calls raise -- there is no CPU
fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .domain import DeviceError, MemplanError, PlanError, SimulationError, TraceError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libstw.so")

STW_OK, STW_ETRACE, STW_EPLAN, STW_ESIM, STW_ECUDA, STW_EARG = range(6)
STW_CAND_FUSION, STW_CAND_GAP = 1, 2
NSTATS = 12
STAT_KEYS = (
    "events", "persistent", "phase_groups", "local_plans", "residual_events", "fusion_attempts",
    "fusion_accepted", "gap_insertions", "layers", "pool_size", "static_peak", "persistent_size",
)


class Batch(C.Structure):
    _fields_ = [
        ("n_traces", C.c_int32), ("on_device", C.c_int32), ("n_events", C.c_int64),
        ("ev_off", C.c_void_p), ("id", C.c_void_p), ("size", C.c_void_p), ("t_s", C.c_void_p),
        ("t_e", C.c_void_p), ("ps", C.c_void_p), ("pe", C.c_void_p), ("dyn", C.c_void_p),
        ("horizon", C.c_void_p), ("n_sched", C.c_void_p),
        ("id32", C.c_void_p), ("size32", C.c_void_p), ("id_base", C.c_int64), ("size_shift", C.c_int32),
        ("reserved", C.c_int32),
    ]


class PlanOpts(C.Structure):
    _fields_ = [("n_cand", C.c_int32), ("select_best", C.c_int32), ("cand", C.c_void_p),
                ("alignment", C.c_int64), ("stream", C.c_void_p)]


class PlanOut(C.Structure):
    _fields_ = [("on_device", C.c_int32)] + [(n, C.c_void_p) for n in (
        "rc", "err_ids", "stats", "addr", "layer_of", "layer_base", "layer_size", "fus_tmp", "fus_avg",
        "order", "best_cand", "addr_best", "best_pool")]


class Report(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "allocated_peak", "reserved_peak", "pool_size", "fallback_count", "fallback_bytes_peak",
        "reuse_hits", "mismatch_count")] + [("efficiency", C.c_double), ("fragmentation", C.c_double)]


class Log(C.Structure):
    _fields_ = [("cap", C.c_int64), ("len", C.c_int64)] + [(n, C.c_void_p) for n in (
        "kind", "t", "id", "size", "addr", "space", "route")]


class Bundle(C.Structure):
    _fields_ = [("pool_size", C.c_int64), ("alignment", C.c_int64), ("n_dec", C.c_int64)] + [
        (n, C.c_void_p) for n in ("d_id", "d_addr", "d_size", "d_ts", "d_te")] + [
        ("n_keys", C.c_int64)] + [(n, C.c_void_p) for n in ("sp_off", "sp_lo", "sp_hi", "key")] + [
        ("reuse", C.c_int32)]


class RectSets(C.Structure):
    _fields_ = [("n_sets", C.c_int32), ("n_cand", C.c_int32), ("n", C.c_int64)] + [
        (n, C.c_void_p) for n in ("set_off", "t_s", "t_e", "size", "addr")]


class LPlans(C.Structure):
    _fields_ = [("n_plans", C.c_int64), ("n", C.c_int64)] + [(n, C.c_void_p) for n in (
        "off", "size", "t_s", "t_e", "addr", "height_in", "t_lo_in", "t_hi_in", "addr_out", "height", "t_lo",
        "t_hi", "tmp", "rc")]


class Fusion(C.Structure):
    _fields_ = [("n_large", C.c_int64), ("n_small", C.c_int64)] + [(n, C.c_void_p) for n in (
        "l_addr", "l_size", "l_ts", "l_te", "s_id", "s_size", "s_ts", "s_te")] + [
        ("l_tmp", C.c_double), ("s_tmp", C.c_double)] + [(n, C.c_int64) for n in (
            "l_height", "l_dur", "s_height", "s_dur")] + [(n, C.c_void_p) for n in (
                "out_addr", "out_order", "result_i", "result_d")]


EXPORTS = (
    "stw_version", "stw_peak_live", "stw_radix_sort_pairs", "stw_plan_batch", "stw_plan_batches", "stw_validate",
    "stw_validate_sets", "stw_reuse_map", "stw_simulate", "stw_baseline", "stw_group_events", "stw_local_plans",
    "stw_weighted_tmp", "stw_fuse_plans", "stw_build_layers", "stw_metrics", "stw_release_scratch", "stw_scan_i64",
)

_lib = None


def load() -> C.CDLL:
    """Load libstw.so (building it first when the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build

    if _build.stale():
        try:
            _build.build()
        except Exception as exc:  # no nvcc on a box that has a prebuilt .so is fine
            if not os.path.exists(LIB_PATH):
                raise DeviceError(f"libstw.so missing and could not be built: {exc}") from exc
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"libstw.so not found at {LIB_PATH}; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    L.stw_version.restype = C.c_char_p
    for name in EXPORTS[1:]:
        if hasattr(L, name):
            getattr(L, name).restype = C.c_int
    L.stw_launch_count.restype = C.c_longlong
    L.stw_prof_enable.restype = None
    L.stw_prof_collect.restype = C.c_int
    _lib = L
    return L


_ERRS = {STW_ETRACE: TraceError, STW_EPLAN: PlanError, STW_ESIM: SimulationError, STW_ECUDA: DeviceError,
         STW_EARG: ValueError}


def check(rc: int, err) -> None:
    if rc == STW_OK:
        return
    msg = err.value.decode(errors="replace") if err is not None else ""
    raise _ERRS.get(rc, MemplanError)(msg or f"libstw error {rc}")


def errbuf():
    return C.create_string_buffer(1024)


def ptr(a):
    """Host numpy array or torch tensor -> c_void_p (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())


def stream_handle(stream=None):
    """cudaStream_t of a torch stream (current stream by default), as void*."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def launch_count() -> int:
    return int(load().stw_launch_count())


def profile(on: bool) -> None:
    load().stw_prof_enable(C.c_int(int(on)))


def profile_collect(reset: bool = True) -> dict:
    """{kernel name: (launches, total device ms)} recorded since the last reset."""
    L = load()
    cap = 256
    names = C.create_string_buffer(64 * cap)
    counts = np.zeros(cap, np.int64)
    ms = np.zeros(cap, np.float64)
    n = L.stw_prof_collect(names, ptr(counts), ptr(ms), C.c_int(cap), C.c_int(int(reset)))
    raw = names.raw
    out = {}
    for i in range(min(n, cap)):
        nm = raw[64 * i: 64 * i + 64].split(b"\0", 1)[0].decode()
        out[nm] = (int(counts[i]), float(ms[i]))
    return out
