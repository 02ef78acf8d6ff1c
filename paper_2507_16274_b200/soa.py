"""Structure-of-arrays trace layout: the contract between the Python API and libstw.

One row per paired event, in the trace's own event order:

    id i64 | size i64 | t_s i32 | t_e i32 | ps i32 | pe i32 | dyn u8 | ls i32 | le i32

`ps`/`pe` are positions in the phase schedule (the ordering the planner uses,
`planner.py:390-392`); a phase absent from the schedule gets an index past
the end and is recorded in `unknown_phase` so that the planner can raise
TraceError exactly where the reference would (`model.py:201-205`). `ls`/`le`
index `layer_names` for dynamic events (-1 for static ones).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .domain import LayerSpan, MemoryRequestEvent, PhaseId, PhaseSpan, TraceError

I32_MAX = np.iinfo(np.int32).max


@dataclass
class TraceArrays:
    id: np.ndarray
    size: np.ndarray
    t_s: np.ndarray
    t_e: np.ndarray
    ps: np.ndarray
    pe: np.ndarray
    dyn: np.ndarray
    ls: np.ndarray
    le: np.ndarray
    phases: list  # PhaseId per schedule slot, then unknown phases
    phase_start: np.ndarray  # schedule spans only
    phase_end: np.ndarray
    layer_names: list
    layer_start: np.ndarray
    layer_end: np.ndarray
    n_known_layers: int = -1  # layer_names past this index are unknown to the schedule
    _dyn_keys: object = field(default=None, repr=False)

    def __len__(self) -> int:
        return int(self.id.shape[0])

    @property
    def n_sched(self) -> int:
        return int(self.phase_start.shape[0])

    @property
    def horizon(self) -> int:
        return int(self.phase_end[-1]) if self.n_sched else 0

    def phase_spans(self):
        return [
            PhaseSpan(self.phases[i], int(self.phase_start[i]), int(self.phase_end[i]))
            for i in range(self.n_sched)
        ]

    def layer_spans(self):
        k = len(self.layer_names) if self.n_known_layers < 0 else self.n_known_layers
        return [
            LayerSpan(n, int(s), int(e))
            for n, s, e in zip(self.layer_names[:k], self.layer_start[:k], self.layer_end[:k])
        ]

    def to_events(self) -> tuple:
        ph, names = self.phases, self.layer_names
        out = []
        cols = zip(
            self.id.tolist(), self.size.tolist(), self.t_s.tolist(), self.t_e.tolist(),
            self.ps.tolist(), self.pe.tolist(), self.dyn.tolist(), self.ls.tolist(),
            self.le.tolist(),
        )
        for i, s, a, b, p, q, d, l1, l2 in cols:
            if d:
                out.append(MemoryRequestEvent(i, s, a, b, ph[p], ph[q], True, names[l1], names[l2]))
            else:
                out.append(MemoryRequestEvent(i, s, a, b, ph[p], ph[q]))
        return tuple(out)

    def static_mask(self) -> np.ndarray:
        return self.dyn == 0

    def dynamic_keys(self):
        """Sorted reuse keys (l_s, l_e) and per-event key index (-1 static).

        Keys sort as string pairs, like `sorted(group_dynamic(...))` (reuse.py:90).
        """
        if self._dyn_keys is None:
            kidx = np.full(len(self), -1, dtype=np.int32)
            d = np.nonzero(self.dyn)[0]
            if d.size == 0:
                self._dyn_keys = ([], kidx)
                return self._dyn_keys
            pairs = self.ls[d].astype(np.int64) * (len(self.layer_names) + 1) + self.le[d]
            uniq, inv = np.unique(pairs, return_inverse=True)
            base = len(self.layer_names) + 1
            keys = [(self.layer_names[u // base], self.layer_names[u % base]) for u in uniq.tolist()]
            order = sorted(range(len(keys)), key=lambda k: keys[k])
            rank = np.empty(len(keys), dtype=np.int32)
            rank[np.asarray(order, dtype=np.int64)] = np.arange(len(keys), dtype=np.int32)
            kidx[d] = rank[inv]
            self._dyn_keys = ([keys[k] for k in order], kidx)
        return self._dyn_keys


def _i32(name: str, values) -> np.ndarray:
    a = np.asarray(values, dtype=np.int64)
    if a.size and (a.min() < 0 or a.max() > I32_MAX):
        raise TraceError(f"{name} outside the supported int32 range")
    return a.astype(np.int32)


def from_trace(trace) -> TraceArrays:
    """Tensorise any trace-like object (this package's or the reference's).

    Duck-typed on the reference attribute names (`model.py:94-124`, `184-199`).
    """
    arr = getattr(trace, "_arrays", None)
    if isinstance(arr, TraceArrays):
        return arr
    return from_events(trace.events, trace.phase_schedule, trace.layer_schedule)


def from_events(events, phase_schedule=(), layer_schedule=()) -> TraceArrays:
    phases = [s.phase for s in phase_schedule]
    index = {}
    for i, p in enumerate(phases):
        index.setdefault(p, i)
    names = [s.name for s in layer_schedule]
    lindex = {}
    for i, n in enumerate(names):
        lindex.setdefault(n, i)
    evs = events if isinstance(events, (list, tuple)) else list(events)
    n = len(evs)

    def pidx(p):
        i = index.get(p)
        if i is None:
            i = index[p] = len(phases)
            phases.append(p)
        return i

    def lidx(name):
        i = lindex.get(name)
        if i is None:  # unknown layer: kept so the reuse stage can raise like the reference
            i = lindex[name] = len(names)
            names.append(name)
        return i

    # one comprehension per attribute (no per-element numpy stores); phase
    # objects are looked up by identity first (a trace reuses a few hundred
    # PhaseId objects), then by value
    by_obj = {}

    def pix(p):
        i = by_obj.get(id(p))
        if i is None:
            i = by_obj[id(p)] = (pidx(p), p)  # (keeps p alive: ids stay unique)
        return i[0]

    ids = [e.id for e in evs]
    sizes = [e.size for e in evs]
    ts = np.array([e.t_s for e in evs], dtype=np.int64)  # (list comprehensions beat generator fromiter ~4x)
    te = np.array([e.t_e for e in evs], dtype=np.int64)
    # phase indices: the distinct phase objects (a trace reuses a few hundred)
    # are collected by identity with C-level maps; when all of them are in the
    # schedule each event's index is one dict lookup, also C-level
    ps_obj = [e.p_s for e in evs]
    pe_obj = [e.p_e for e in evs]
    uniq = dict(zip(map(id, ps_obj), ps_obj))
    uniq.update(zip(map(id, pe_obj), pe_obj))
    if all(p in index for p in uniq.values()):
        idmap = {k: index[p] for k, p in uniq.items()}
        ps = np.array(list(map(idmap.__getitem__, map(id, ps_obj))), dtype=np.int32)
        pe = np.array(list(map(idmap.__getitem__, map(id, pe_obj))), dtype=np.int32)
    else:
        # p_s then p_e of each event in turn: phases missing from the schedule
        # get their indices in the reference's order of first appearance
        pp = np.fromiter((pix(x) for e in evs for x in (e.p_s, e.p_e)), dtype=np.int32, count=2 * n)
        ps, pe = np.ascontiguousarray(pp[0::2]), np.ascontiguousarray(pp[1::2])
    del ps_obj, pe_obj, uniq
    dyn = np.array([e.dynamic for e in evs], dtype=bool).view(np.uint8)
    ls = np.full(n, -1, dtype=np.int32)
    le = np.full(n, -1, dtype=np.int32)
    for k in np.flatnonzero(dyn).tolist():
        ls[k] = lidx(evs[k].l_s)
        le[k] = lidx(evs[k].l_e)
    try:
        id_arr = np.asarray(ids, dtype=np.int64)
        size_arr = np.asarray(sizes, dtype=np.int64)
    except OverflowError:
        raise TraceError("event id or size outside the supported int64 range") from None
    nl = len(layer_schedule)
    return TraceArrays(
        id=id_arr,
        size=size_arr,
        t_s=_i32("t_s", ts),
        t_e=_i32("t_e", te),
        ps=ps,
        pe=pe,
        dyn=dyn,
        ls=ls,
        le=le,
        phases=phases,
        phase_start=np.asarray([s.start for s in phase_schedule], dtype=np.int64),
        phase_end=np.asarray([s.end for s in phase_schedule], dtype=np.int64),
        layer_names=names,
        layer_start=np.asarray([s.start for s in layer_schedule] + [0] * (len(names) - nl), dtype=np.int64),
        layer_end=np.asarray([s.end for s in layer_schedule] + [-1] * (len(names) - nl), dtype=np.int64),
        n_known_layers=nl,
    )
