"""One large trace over several GPUs.

The planner greedy itself has no partition (replicas only); its three
data-parallel checks split across ranks with one small exchange each:

* K7 `validate_plan` (planner.py:476-505). The reference sweep's report for
  decision d depends only on the decisions allocated before d that are still
  live at t_s(d), inserted in sweep order ((t_s, id), frees first at equal t).
  The (t_s, id)-sorted decisions are cut into `world` contiguous bands; rank r
  validates its band together with the band's halo -- the earlier decisions
  still live at the band's first start -- and keeps the pairs whose second
  (reporting) decision lies in its band. Those are exactly the reference's
  pairs for the band, in its order, so the rank-ordered concatenation
  (allgather) is the reference's list.
* K1 `peak_live_bytes` (model.py:261-276). The timeline is cut into `world`
  bands at quantiles of t_s. Clipping every event to a band leaves live(t)
  unchanged inside it, so the peak is the allreduce MAX of the band peaks.
* K8 reusable spaces (reuse.py:54-93). Keys are dealt round-robin and the
  interval lists allgathered back into key order.

Every function takes the per-band worker as an argument (default: the device
kernels through `api`) so the decomposition itself can be checked on CPU
against the oracle. Collectives go through torch.distributed (NCCL on GPUs,
gloo in the CPU tests)."""

from __future__ import annotations

import numpy as np

from .plan_types import DecisionColumns, ReuseEntry, ReuseMap


def _dist():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def allgather_rows(local: np.ndarray, device=None) -> list:
    """Every rank's int64 [k_r, w] array, in rank order (variable k_r)."""
    import torch
    import torch.distributed as dist

    local = np.ascontiguousarray(local, np.int64)
    _, world = _dist()
    if world == 1:
        return [local]
    w = local.shape[1]
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    counts = [int(x.item()) for x in ns]
    m = max(max(counts), 1)
    buf = torch.zeros((m, w), dtype=torch.int64, device=device)
    buf[: local.shape[0]] = torch.from_numpy(local).to(buf.device)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    return [o[:c].cpu().numpy() for o, c in zip(outs, counts)]


def _allreduce_max(v: int, device=None) -> int:
    import torch
    import torch.distributed as dist

    _, world = _dist()
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return int(t.item())


# ---------------------------------------------------------------- K7
def sweep_order(cols: DecisionColumns) -> np.ndarray:
    """Allocation order of the reference sweep: (t_s, id)."""
    return np.lexsort((cols.id, cols.t_s))


def band_rows(cols: DecisionColumns, rank: int, world: int, order=None):
    """Rows rank `rank` validates: (halo rows, band rows), both in sweep order."""
    n = len(cols)
    order = sweep_order(cols) if order is None else order
    r0, r1 = n * rank // world, n * (rank + 1) // world
    if r0 >= r1:
        return order[:0], order[:0]
    pre = order[:r0]
    halo = pre[cols.t_e[pre] > cols.t_s[order[r0]]]
    return halo, order[r0:r1]


def validate_band(cols: DecisionColumns, rank: int, world: int, validate=None, order=None) -> np.ndarray:
    """The reference report's pairs whose reporting decision is in band `rank`,
    as row indices [k, 2], in the reference's order."""
    if validate is None:
        from .api import validate_columns as validate
    halo, band = band_rows(cols, rank, world, order)
    if band.size == 0:
        return np.zeros((0, 2), np.int64)
    sub = np.concatenate([halo, band])
    pairs = np.asarray(validate(cols.id[sub], cols.addr[sub], cols.size[sub], cols.t_s[sub], cols.t_e[sub]),
                       np.int64).reshape(-1, 2)
    mine = pairs[pairs[:, 1] >= halo.size]
    return sub[mine]


def validate_plan_sharded(plan, validate=None, device=None) -> list:
    """`validate_plan` of one plan, each rank sweeping one band (+ halo)."""
    from .plan_types import StaticPlan

    if isinstance(plan, StaticPlan):
        cols, decs = plan.columns(), plan.decisions
    else:
        decs = tuple(plan.decisions)
        cols = DecisionColumns.from_decisions(decs)
    rank, world = _dist()
    local = validate_band(cols, rank, world, validate)
    rows = np.concatenate(allgather_rows(local, device))
    return [(decs[a], decs[b]) for a, b in rows.tolist()]


# ---------------------------------------------------------------- K1
def time_bands(t_s: np.ndarray, world: int) -> np.ndarray:
    """world + 1 band edges at quantiles of t_s (first -inf, last +inf)."""
    ts = np.sort(np.asarray(t_s, np.int64))
    n = ts.size
    edges = np.empty(world + 1, np.int64)
    edges[0], edges[world] = np.iinfo(np.int64).min, np.iinfo(np.int64).max
    for r in range(1, world):
        edges[r] = ts[min(n * r // world, n - 1)] if n else 0
    return edges


def peak_band(size, t_s, t_e, rank: int, world: int, peak=None) -> int:
    """Peak live bytes inside time band `rank` (events clipped to it)."""
    if peak is None:
        from .api import peak_live_columns as peak
    t_s = np.asarray(t_s, np.int64)
    t_e = np.asarray(t_e, np.int64)
    e = time_bands(t_s, world)
    a, b = e[rank], e[rank + 1]
    m = (t_s < b) & (t_e > a)
    if not m.any():
        return 0
    return int(peak(np.asarray(size, np.int64)[m], np.maximum(t_s[m], a), np.minimum(t_e[m], b)))


def peak_live_bytes_sharded(events, peak=None, device=None) -> int:
    """`peak_live_bytes` (model.py:261-276) with the timeline split over ranks."""
    ev = list(events)
    size = np.asarray([x.size for x in ev], np.int64)
    ts = np.asarray([x.t_s for x in ev], np.int64)
    te = np.asarray([x.t_e for x in ev], np.int64)
    rank, world = _dist()
    return _allreduce_max(peak_band(size, ts, te, rank, world, peak), device)


# ---------------------------------------------------------------- K8
def reuse_keys_of(rank: int, world: int, n_keys: int) -> np.ndarray:
    return np.arange(rank, n_keys, world, dtype=np.int64)


def reuse_rows(plan, trace, rank: int, world: int, spaces=None):
    """Keys, windows and this rank's (key, lo, hi) idle intervals [k, 3]."""
    from . import api

    if spaces is None:
        spaces = api.reusable_spaces
    ta = getattr(trace, "_arrays", None)
    keys = ta.dynamic_keys()[0] if ta is not None else sorted(api.group_dynamic(trace.dynamic_events()))
    if not keys:
        return keys, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 3), np.int64)
    t_lo, t_hi = api._windows(keys, trace.layer_schedule)
    mine = reuse_keys_of(rank, world, len(keys))
    got = spaces(api._plan_columns(plan), t_lo[mine], t_hi[mine]) if mine.size else []
    rows = [(int(k), iv.lo, iv.hi) for k, s in zip(mine.tolist(), got) for iv in s]
    return keys, t_lo, t_hi, np.asarray(rows, np.int64).reshape(-1, 3)


def assemble_reuse_map(keys, t_lo, t_hi, rows: np.ndarray) -> ReuseMap:
    """ReuseMap in key order from every rank's rows (keys with no rows: empty)."""
    from .ivset import IntervalSet

    per = {k: ([], []) for k in range(len(keys))}
    for k, lo, hi in np.asarray(rows, np.int64).reshape(-1, 3).tolist():
        per[k][0].append(lo)
        per[k][1].append(hi)
    return ReuseMap({keys[k]: ReuseEntry(int(t_lo[k]), int(t_hi[k]),
                                         IntervalSet.from_bounds(per[k][0], per[k][1]))
                     for k in range(len(keys))})


def derive_reuse_map_sharded(plan, trace, spaces=None, device=None) -> ReuseMap:
    """`derive_reuse_map` (reuse.py:83-93) with the keys dealt over ranks."""
    rank, world = _dist()
    keys, t_lo, t_hi, rows = reuse_rows(plan, trace, rank, world, spaces)
    if not keys:
        return ReuseMap({})
    return assemble_reuse_map(keys, t_lo, t_hi, np.concatenate(allgather_rows(rows, device)))
