"""The reference planner module's API (`memplan/planner.py`), sub-operations
included: grouping, packing, TMP, fusion, layers, global planning, validation.

Every computation is a libstw call (include/stw.h, "sub-operations"):
`group_by_phase` -> stw_group_events, `pack_group` / `_plan_from_decisions` /
`compute_tmp` -> stw_local_plans, `weighted_tmp_average` -> stw_weighted_tmp,
`fuse_plans` / `try_fuse` -> stw_fuse_plans, `build_layers_for_size` ->
stw_build_layers; `synthesize_static_plan` / `validate_plan` are the batched
planner and K7 (api.py). Python only marshals the reference's value objects
(`HomoPhaseGroup`, `LocalPlan`, `MemoryLayer`, `_Item`) to columns and back.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence, Union

import numpy as np

from . import _lib
from .api import synthesize_static_plan, validate_plan
from .domain import AllocationDecision, MemoryRequestEvent, PhaseId, PlanError
from .plan_types import MemoryLayer, PlanStats, StaticPlan, _Keyed

GroupKey = tuple  # (PhaseId, PhaseId)

__all__ = [
    "GroupKey", "HomoPhaseGroup", "LocalPlan", "MemoryLayer", "PlanStats", "StaticPlan", "build_layers_for_size",
    "compute_tmp", "fuse_plans", "group_by_phase", "pack_group", "pack_groups", "synthesize_static_plan", "try_fuse",
    "validate_plan", "weighted_tmp_average",
]


@dataclass(frozen=True)
class HomoPhaseGroup:
    """Static requests sharing one (alloc phase, free phase) pair (planner.py:41-50)."""

    key: GroupKey
    members: tuple

    @property
    def cross_phase(self) -> bool:
        return self.key[0] != self.key[1]


@dataclass(frozen=True)
class LocalPlan:
    """A packed group: decisions with group-relative addresses (planner.py:53-71)."""

    key: GroupKey
    decisions: tuple
    height: int
    t_s: int
    t_e: int
    tmp: float

    @property
    def duration(self) -> int:
        return self.t_e - self.t_s

    @property
    def space_time(self) -> int:
        """Denominator of the occupancy ratio; the fusion acceptance weight."""
        return self.height * self.duration


@dataclass(frozen=True)
class _Item:
    """One layer occupant candidate: a residual event or a local plan (planner.py:225-233)."""

    size: int
    t_s: int
    t_e: int
    tie: int
    payload: Union[MemoryRequestEvent, LocalPlan, None]


def _i64(values) -> np.ndarray:
    return np.ascontiguousarray(np.fromiter(values, dtype=np.int64), dtype=np.int64)


def _phase_code(p: PhaseId) -> int:
    """PhaseId order (kind, microbatch, chunk) as one int64."""
    if p.microbatch >= 1 << 30 or p.chunk >= 1 << 30:
        raise ValueError(f"phase {p} out of range for the device key")
    return (int(p.kind) << 60) | (p.microbatch << 30) | p.chunk


# ---------------------------------------------------------------------------
# grouping


def group_by_phase(events: Iterable[MemoryRequestEvent]) -> list:
    """Partition static events by (p_s, p_e); members sorted by (t_s, id);
    groups in (p_s, p_e) order (planner.py:74-85)."""
    evs = list(events)
    for ev in evs:
        if ev.dynamic:
            raise PlanError(f"event {ev.id} is dynamic; phase groups hold static only")
    n = len(evs)
    if n == 0:
        return []
    ps = _i64(_phase_code(e.p_s) for e in evs)
    pe = _i64(_phase_code(e.p_e) for e in evs)
    ts = _i64(e.t_s for e in evs)
    ids = _i64(e.id for e in evs)
    perm = np.empty(n, np.int32)
    off = np.empty(n + 1, np.int64)
    ng = C.c_int64(0)
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_group_events(C.c_int64(n), _lib.ptr(ps), _lib.ptr(pe), _lib.ptr(ts), _lib.ptr(ids),
                                            _lib.ptr(perm), _lib.ptr(off), C.byref(ng), None, err, C.sizeof(err)), err)
    out = []
    p = perm.tolist()
    for g in range(ng.value):
        members = tuple(evs[i] for i in p[off[g]:off[g + 1]])
        out.append(HomoPhaseGroup((members[0].p_s, members[0].p_e), members))
    return out


# ---------------------------------------------------------------------------
# packing and the time-memory product


def _local_plans(member_lists, addrs=None, overrides=None):
    """One stw_local_plans call over several member lists; returns per plan
    (relative addresses or None, height, t_lo, t_hi, tmp, rc)."""
    P = len(member_lists)
    off = np.zeros(P + 1, np.int64)
    off[1:] = np.cumsum([len(m) for m in member_lists])
    flat = [d for m in member_lists for d in m]
    n = len(flat)
    size = _i64(d.size for d in flat)
    ts = _i64(d.t_s for d in flat)
    te = _i64(d.t_e for d in flat)
    addr = _i64(d.addr for d in flat) if addrs == "given" else None
    addr_out = np.empty(max(n, 1), np.int64) if addr is None else None
    h_in = lo_in = hi_in = None
    if overrides is not None:
        h_in, lo_in, hi_in = (_i64(x) for x in zip(*overrides))
    height = np.empty(P, np.int64)
    t_lo = np.empty(P, np.int64)
    t_hi = np.empty(P, np.int64)
    tmp = np.empty(P, np.float64)
    rc = np.empty(P, np.int32)
    lp = _lib.LPlans(P, n, *(_lib.ptr(x) for x in (off, size, ts, te, addr, h_in, lo_in, hi_in, addr_out, height,
                                                   t_lo, t_hi, tmp, rc)))
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_local_plans(C.byref(lp), None, err, C.sizeof(err)), err)
    res = []
    for p in range(P):
        rel = addr_out[off[p]:off[p + 1]].tolist() if addr_out is not None else None
        res.append((rel, int(height[p]), int(t_lo[p]), int(t_hi[p]), float(tmp[p]), int(rc[p])))
    return res


def _check_tmp_rc(key, rc: int) -> None:
    if rc == _lib.STW_EPLAN:
        raise PlanError(f"group {key}: degenerate lifespan")
    if rc != _lib.STW_OK:
        raise ZeroDivisionError("division by zero")


def pack_groups(groups: Sequence[HomoPhaseGroup]) -> list:
    """pack_group of many groups in one device call."""
    for g in groups:
        if not g.members:
            raise PlanError("cannot pack an empty group")
    if not groups:
        return []
    out = []
    for g, (rel, h, lo, hi, tmp, rc) in zip(groups, _local_plans([g.members for g in groups])):
        _check_tmp_rc(g.key, rc)
        out.append(LocalPlan(g.key, tuple(AllocationDecision(ev, a) for ev, a in zip(g.members, rel)), h, lo, hi,
                             tmp))
    return out


def pack_group(group: HomoPhaseGroup) -> LocalPlan:
    """Stack the group contiguously in member order (prefix sums; planner.py:98-107)."""
    return pack_groups([group])[0]


def _plan_from_decisions(key, decisions: Sequence[AllocationDecision]) -> LocalPlan:
    """Height, span and TMP of decisions with given addresses (planner.py:88-95)."""
    decisions = tuple(decisions)
    if not decisions:
        raise ValueError("max() arg is an empty sequence")
    (_, h, lo, hi, tmp, rc), = _local_plans([decisions], addrs="given")
    _check_tmp_rc(key, rc)
    return LocalPlan(key, decisions, h, lo, hi, tmp)


def compute_tmp(plan: LocalPlan) -> float:
    """Occupancy of the plan's space-time rectangle, in (0, 1] (planner.py:110-115)."""
    if plan.t_e <= plan.t_s:
        raise PlanError(f"group {plan.key}: degenerate lifespan")
    (_, _h, _lo, _hi, tmp, rc), = _local_plans([plan.decisions], addrs="given",
                                                overrides=[(plan.height, plan.t_s, plan.t_e)])
    _check_tmp_rc(plan.key, rc)
    return tmp


def weighted_tmp_average(plans: Sequence[LocalPlan]) -> float:
    """Occupancies weighted by space-time area, CPython float semantics (planner.py:118-121)."""
    plans = list(plans)
    if not plans:
        raise ZeroDivisionError("division by zero")
    if sum(p.space_time for p in plans) == 0:
        raise ZeroDivisionError("float division by zero")
    tmp = np.asarray([float(p.tmp) for p in plans], np.float64)
    h = _i64(p.height for p in plans)
    d = _i64(p.duration for p in plans)
    out = C.c_double(0.0)
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_weighted_tmp(C.c_int64(len(plans)), _lib.ptr(tmp), _lib.ptr(h), _lib.ptr(d),
                                            C.byref(out), None, err, C.sizeof(err)), err)
    return out.value


# ---------------------------------------------------------------------------
# fusion


def _fuse(larger: LocalPlan, smaller: LocalPlan):
    L, S = larger.decisions, smaller.decisions
    la = _i64(d.addr for d in L)
    ls = _i64(d.size for d in L)
    lts = _i64(d.t_s for d in L)
    lte = _i64(d.t_e for d in L)
    sid = _i64(d.id for d in S)
    ss = _i64(d.size for d in S)
    sts = _i64(d.t_s for d in S)
    ste = _i64(d.t_e for d in S)
    out_addr = np.empty(len(S), np.int64)
    out_order = np.empty(len(S), np.int32)
    ri = np.zeros(4, np.int64)
    rd = np.zeros(2, np.float64)
    fz = _lib.Fusion(len(L), len(S), *(_lib.ptr(x) for x in (la, ls, lts, lte, sid, ss, sts, ste)),
                     float(larger.tmp), float(smaller.tmp), int(larger.height), int(larger.duration),
                     int(smaller.height), int(smaller.duration),
                     *(_lib.ptr(x) for x in (out_addr, out_order, ri, rd)))
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_fuse_plans(C.byref(fz), None, err, C.sizeof(err)), err)
    key = ((larger if larger.t_s <= smaller.t_s else smaller).key[0],
           (larger if larger.t_e >= smaller.t_e else smaller).key[1])
    _check_tmp_rc(key, int(ri[3]))
    placed = tuple(AllocationDecision(S[i].event, int(out_addr[i])) for i in out_order.tolist())
    fused = LocalPlan(key, tuple(L) + placed, int(ri[0]), int(ri[1]), int(ri[2]), float(rd[0]))
    return fused, float(rd[1])


def fuse_plans(larger: LocalPlan, smaller: LocalPlan) -> LocalPlan:
    """Insert the smaller plan's requests into the larger plan by the cursor walk
    (planner.py:132-169)."""
    if not smaller.decisions:
        return larger
    if not larger.decisions:
        return smaller
    return _fuse(larger, smaller)[0]


def try_fuse(larger: LocalPlan, smaller: LocalPlan) -> Optional[LocalPlan]:
    """Fuse; keep the result only if its TMP strictly beats the space-time
    weighted average of the two (planner.py:172-182)."""
    if not smaller.decisions:
        return larger
    if not larger.decisions:
        return smaller
    if larger.space_time + smaller.space_time == 0:
        raise ZeroDivisionError("float division by zero")
    fused, avg = _fuse(larger, smaller)
    return fused if fused.tmp > avg else None


# ---------------------------------------------------------------------------
# memory layers


def _as_double(v, what: str) -> float:
    if isinstance(v, (int, np.integer)) and abs(int(v)) >= 1 << 53:
        raise ValueError(f"{what} {v} beyond exact double range")
    return float(v)


def build_layers_for_size(items: Sequence[_Item]) -> list:
    """Alg. 1 for one size class (planner.py:236-254): items in (t_s, tie) order
    join the layer whose end is the largest one strictly below their start
    (ties: oldest), else open a new layer."""
    items = list(items)
    n = len(items)
    if n == 0:
        return []
    ts = np.asarray([_as_double(i.t_s, "t_s") for i in items], np.float64)
    te = np.asarray([_as_double(i.t_e, "t_e") for i in items], np.float64)
    tie = _i64(i.tie for i in items)
    layer_of = np.empty(n, np.int32)
    order = np.empty(n, np.int32)
    nl = C.c_int64(0)
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_build_layers(C.c_int64(n), _lib.ptr(ts), _lib.ptr(te), _lib.ptr(tie),
                                            _lib.ptr(layer_of), _lib.ptr(order), C.byref(nl), None, err,
                                            C.sizeof(err)), err)
    layers: list = []
    for k in order.tolist():
        it = items[k]
        li = int(layer_of[k])
        if li == len(layers):
            layers.append(MemoryLayer(size=it.size))
        layers[li].insert(it.t_s, it.t_e, it.payload)
    if len(layers) != nl.value:
        raise RuntimeError("layer count mismatch between device and host")
    return layers


# the reference's private helpers, for code that imports them
__all__ += ["_Item", "_Keyed", "_plan_from_decisions"]
