"""Planner value objects mirroring the reference (`planner.py:41-71`, `189-326`).

`StaticPlan` built by the device path keeps the columnar result (ids,
addresses, sizes, lifespans in (t_s, id) order) and materialises the
reference's `AllocationDecision` tuple only when `.decisions` is read, so
array consumers (the replay scorer, the batched sweep) never pay for objects.
"""

from __future__ import annotations

from bisect import bisect_left
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .domain import AllocationDecision
from .ivset import IntervalSet


@dataclass
class PlanStats:
    """Planner counters (planner.py:261-294)."""

    num_events: int = 0
    num_persistent: int = 0
    num_groups: int = 0
    num_plans: int = 0
    num_residuals: int = 0
    fusion_attempts: int = 0
    fusion_accepted: int = 0
    gap_insertions: int = 0
    num_layers: int = 0
    pool_size: int = 0
    static_peak: int = 0
    plan_seconds: float = 0.0
    accepted_fusions: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {
            "events": self.num_events,
            "persistent": self.num_persistent,
            "phase_groups": self.num_groups,
            "local_plans": self.num_plans,
            "residual_events": self.num_residuals,
            "fusion_attempts": self.fusion_attempts,
            "fusion_accepted": self.fusion_accepted,
            "gap_insertions": self.gap_insertions,
            "layers": self.num_layers,
            "pool_size": self.pool_size,
            "static_peak": self.static_peak,
            "plan_seconds": self.plan_seconds,
        }


class _Keyed:
    """Opaque slot payload holder (planner.py:215-222): slots compare by their
    lifespans only, the payload rides along as `.value`."""

    __slots__ = ("value",)

    def __init__(self, value):
        self.value = value

    def __repr__(self) -> str:
        return f"_Keyed({self.value!r})"


class MemoryLayer:
    """A size-S address band time-shared by lifespan-disjoint occupants
    (planner.py:189-212). `slots` holds (t_s, t_e, _Keyed(payload)) sorted by
    start; `end` is the largest t_e inserted. Layers of a device plan fill
    their slots lazily from the plan's columns, one slot per member event."""

    __slots__ = ("size", "base", "end", "_slots", "_starts", "_slots_fn")

    def __init__(self, size: int, slots=None, end: int = -1, base: Optional[int] = None, *, slots_fn=None):
        self.size = size
        self.base = base
        self.end = end
        self._slots = list(slots) if slots is not None else (None if slots_fn else [])
        self._starts = None
        self._slots_fn = slots_fn

    @property
    def slots(self) -> list:
        if self._slots is None:
            self._slots = self._slots_fn()
        return self._slots

    def _starts_list(self) -> list:
        if self._starts is None or len(self._starts) != len(self.slots):
            self._starts = [s[0] for s in self.slots]
        return self._starts

    def fits_gap(self, t_s, t_e) -> bool:
        """True iff [t_s, t_e] (closed) touches no slot (planner.py:199-205)."""
        starts = self._starts_list()
        i = bisect_left(starts, t_s)
        if i and self.slots[i - 1][1] >= t_s:
            return False
        return not (i < len(starts) and starts[i] <= t_e)

    def insert(self, t_s, t_e, payload) -> None:
        """Add an occupant, keeping slots sorted by start (planner.py:207-212)."""
        starts = self._starts_list()
        i = bisect_left(starts, t_s)
        starts.insert(i, t_s)
        self.slots.insert(i, (t_s, t_e, _Keyed(payload)))
        if t_e > self.end:
            self.end = t_e

    def __eq__(self, other):
        if not isinstance(other, MemoryLayer):
            return NotImplemented
        return (self.size, self.end, self.base, [s[:2] for s in self.slots]) == (
            other.size, other.end, other.base, [s[:2] for s in other.slots])

    __hash__ = None

    def __repr__(self) -> str:
        return f"MemoryLayer(size={self.size}, base={self.base}, end={self.end})"


@dataclass(frozen=True)
class PlanDecision:
    """File-shaped decision (traceio.py:298-310)."""

    id: int
    addr: int
    size: int
    t_s: int
    t_e: int

    @property
    def interval(self):
        from .ivset import Interval

        return Interval(self.addr, self.addr + self.size)


@dataclass(frozen=True)
class PlanBundle:
    """What the replay scorer needs from a plan (traceio.py:313-331)."""

    pool_size: int
    alignment: int
    decisions: tuple
    reuse: dict

    def validate(self) -> None:
        from .domain import PlanError

        for d in self.decisions:
            if d.addr < 0 or d.addr + d.size > self.pool_size:
                raise PlanError(f"decision {d.id} out of pool")
            if d.addr % self.alignment:
                raise PlanError(f"decision {d.id} misaligned address {d.addr}")
        for key, space in self.reuse.items():
            for iv in space:
                if iv.lo < 0 or iv.hi > self.pool_size:
                    raise PlanError(f"reuse entry {key} outside pool")


class DecisionColumns:
    """Columnar decisions in (t_s, id) order: id, addr, size, t_s, t_e (+ source index)."""

    __slots__ = ("id", "addr", "size", "t_s", "t_e", "src")

    def __init__(self, id, addr, size, t_s, t_e, src=None):
        self.id = np.ascontiguousarray(id, dtype=np.int64)
        self.addr = np.ascontiguousarray(addr, dtype=np.int64)
        self.size = np.ascontiguousarray(size, dtype=np.int64)
        self.t_s = np.ascontiguousarray(t_s, dtype=np.int32)
        self.t_e = np.ascontiguousarray(t_e, dtype=np.int32)
        self.src = src

    def __len__(self) -> int:
        return int(self.id.shape[0])

    @classmethod
    def from_decisions(cls, decisions) -> "DecisionColumns":
        n = len(decisions)
        cols = np.empty((5, n), dtype=object)
        for k, d in enumerate(decisions):
            cols[0, k], cols[1, k], cols[2, k], cols[3, k], cols[4, k] = d.id, d.addr, d.size, d.t_s, d.t_e
        return cls(cols[0].astype(np.int64), cols[1].astype(np.int64), cols[2].astype(np.int64),
                   cols[3].astype(np.int64), cols[4].astype(np.int64))


class StaticPlan:
    """The planner's output (planner.py:297-326)."""

    __slots__ = ("pool_size", "alignment", "_decisions", "_layer_table", "persistent_size", "_cols", "_events",
                 "_layer_fn")

    def __init__(self, pool_size, alignment, decisions=(), layer_table=(), persistent_size=0):
        self.pool_size = pool_size
        self.alignment = alignment
        self._decisions = tuple(decisions)
        self._layer_table = tuple(layer_table)
        self.persistent_size = persistent_size
        self._cols = None
        self._events = None
        self._layer_fn = None

    @classmethod
    def from_columns(cls, pool_size, alignment, cols: DecisionColumns, events_fn, persistent_size, layer_fn=None):
        p = cls(pool_size, alignment, (), (), persistent_size)
        p._decisions = None
        p._layer_table = None
        p._cols = cols
        p._events = events_fn
        p._layer_fn = layer_fn
        return p

    @property
    def decisions(self) -> tuple:
        if self._decisions is None:
            events = self._events()
            self._decisions = tuple(
                AllocationDecision(events[s], a) for s, a in zip(self._cols.src.tolist(), self._cols.addr.tolist())
            )
        return self._decisions

    @property
    def layer_table(self) -> tuple:
        if self._layer_table is None:
            self._layer_table = self._layer_fn() if self._layer_fn else ()
        return self._layer_table

    def columns(self) -> DecisionColumns:
        if self._cols is None:
            self._cols = DecisionColumns.from_decisions(self._decisions)
        return self._cols

    def address_span(self) -> IntervalSet:
        """[min addr, max end) of the plan (planner.py:307-313)."""
        c = self.columns()
        if len(c) == 0:
            return IntervalSet.empty()
        return IntervalSet.span(int(c.addr.min()), int((c.addr + c.size).max()))

    def to_bundle(self, reuse=None) -> PlanBundle:
        rcols = getattr(reuse, "_cols", None)  # the device's reuse columns (derive_reuse_map)
        if hasattr(reuse, "spaces"):
            reuse = reuse.spaces()
        c = self.columns()
        decs = tuple(
            PlanDecision(i, a, s, ts, te)
            for i, a, s, ts, te in zip(c.id.tolist(), c.addr.tolist(), c.size.tolist(), c.t_s.tolist(), c.t_e.tolist())
        )
        b = PlanBundle(self.pool_size, self.alignment, decs, dict(reuse or {}))
        object.__setattr__(b, "_cols", c)
        if rcols is not None:
            object.__setattr__(b, "_reuse_cols", rcols)
        return b

    def __eq__(self, other):
        if not isinstance(other, StaticPlan):
            return NotImplemented
        return (self.pool_size, self.alignment, self.persistent_size, self.decisions) == (
            other.pool_size, other.alignment, other.persistent_size, other.decisions)

    __hash__ = None

    def __repr__(self) -> str:
        return f"StaticPlan(pool_size={self.pool_size}, decisions=<{len(self.columns())}>)"


@dataclass(frozen=True)
class ReuseEntry:
    """Reusable space of one dynamic (alloc layer, free layer) group (reuse.py:21-25)."""

    t_lo: int
    t_hi: int
    space: IntervalSet


@dataclass(frozen=True)
class ReuseMap:
    """One entry per dynamic reuse key, keys in sorted order (reuse.py:28-39)."""

    entries: dict

    def spaces(self) -> dict:
        return {key: entry.space for key, entry in self.entries.items()}

    def __contains__(self, key) -> bool:
        return key in self.entries

    def get(self, key):
        return self.entries.get(key)


@dataclass(frozen=True)
class SimReport:
    """Replay outcome (sim.py:39-64)."""

    allocated_peak: int
    reserved_peak: int
    efficiency: float
    fragmentation: float
    pool_size: int
    fallback_count: int
    fallback_bytes_peak: int
    reuse_hits: int
    mismatch_count: int

    def to_dict(self) -> dict:
        return {
            "allocated_peak": self.allocated_peak,
            "reserved_peak": self.reserved_peak,
            "efficiency": self.efficiency,
            "fragmentation": self.fragmentation,
            "pool_size": self.pool_size,
            "fallback_count": self.fallback_count,
            "fallback_bytes_peak": self.fallback_bytes_peak,
            "reuse_hits": self.reuse_hits,
            "mismatch_count": self.mismatch_count,
        }
