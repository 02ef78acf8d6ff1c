"""Host-side logic (no device): domain types, SoA tensorisation, interval
algebra (bitmap oracle, as test_intervals.py:13-21 does), plan files."""

import random

import numpy as np
import pytest

from paper_2507_16274_b200 import api, planio, soa, tracegen
from paper_2507_16274_b200.domain import (MemoryRequestEvent, PhaseId, PhaseKind, PhaseSpan, PlanError, Trace,
                                          TraceError, align_up)
from paper_2507_16274_b200.ivset import Interval, IntervalSet, best_fit, intersect, subtract
from paper_2507_16274_b200.plan_types import PlanBundle, PlanDecision

U = 128


def bits(s):
    out = set()
    for iv in s:
        out.update(range(iv.lo, iv.hi))
    return out


def from_bits(b):
    return IntervalSet(Interval(x, x + 1) for x in b)


def rand_set(rng):
    return IntervalSet(Interval(a, a + rng.randint(1, 24)) for a in (rng.randint(0, U - 1) for _ in range(rng.randint(0, 12))))


def test_intervalset_algebra_matches_bitmap_oracle():
    rng = random.Random(0)
    for _ in range(500):
        x, y = rand_set(rng), rand_set(rng)
        for s in (x, y):
            ivs = s.intervals
            assert all(a.hi < b.lo for a, b in zip(ivs, ivs[1:]))
        assert bits(intersect(x, y)) == bits(x) & bits(y)
        assert bits(subtract(x, y)) == bits(x) - bits(y)
        assert bits(x.union(y)) == bits(x) | bits(y)
        a = rng.randint(0, U - 2)
        iv = Interval(a, a + rng.randint(1, 10))
        assert bits(x.add(iv)) == bits(x) | set(range(iv.lo, iv.hi))
        assert bits(x.remove(iv)) == bits(x) - set(range(iv.lo, iv.hi))
        assert x.add(iv) == from_bits(bits(x) | set(range(iv.lo, iv.hi)))
        assert x.contains_interval(iv) == any(v.contains(iv) for v in x)
        size = rng.randint(1, 12)
        cands = [v for v in x if v.length >= size]
        want = min(cands, key=lambda v: (v.length, v.lo)) if cands else None
        assert best_fit(x, size) == want


def test_intervalset_spec_examples():
    s = IntervalSet([Interval(0, 10), Interval(10, 20), Interval(5, 12)])  # test_intervals.py:46-49
    assert s.intervals == (Interval(0, 20),)
    x = IntervalSet([Interval(0, 50), Interval(80, 100)])
    assert intersect(x, IntervalSet([Interval(30, 90)])) == IntervalSet([Interval(30, 50), Interval(80, 90)])
    with pytest.raises(ValueError):
        Interval(5, 5)
    with pytest.raises(ValueError):
        best_fit(x, 0)


def test_phase_tags_and_events():
    for tag in ("init", "opt", "F:0", "B:3", "F:2.1", "B:12.7"):  # test_model.py:25-27
        assert PhaseId.parse(tag).tag() == tag
    for bad in ("X:1", "F:", "forward", "F:1.2.3", ""):
        with pytest.raises(TraceError):
            PhaseId.parse(bad)
    with pytest.raises(ValueError):
        PhaseId(PhaseKind.INIT, microbatch=2)
    assert (align_up(1), align_up(512), align_up(513)) == (512, 512, 1024)
    F, B = PhaseId.parse("F:0"), PhaseId.parse("B:0")
    with pytest.raises(TraceError):
        MemoryRequestEvent(0, 0, 0, 5, F, B)
    with pytest.raises(TraceError):
        MemoryRequestEvent(0, 512, 5, 5, F, B)
    with pytest.raises(TraceError):
        MemoryRequestEvent(0, 512, 0, 5, F, B, dynamic=True)
    with pytest.raises(TraceError):
        MemoryRequestEvent(0, 512, 0, 5, F, B, l_s="a", l_e="b")


def test_soa_round_trip_and_lazy_trace():
    ta = tracegen.synth_arrays(tracegen.SynthConfig.for_preset("moe_recompute", seed=3))
    tr = Trace.from_arrays(ta)
    tr.validate()
    tb = soa.from_events(tr.events, tr.phase_schedule, tr.layer_schedule)
    for f in ("id", "size", "t_s", "t_e", "ps", "pe", "dyn", "ls", "le"):
        assert np.array_equal(getattr(ta, f), getattr(tb, f)), f
    assert Trace(tr.events, tr.phase_schedule, tr.layer_schedule) == tr
    keys, kidx = ta.dynamic_keys()
    assert keys == sorted(api.group_dynamic(tr.dynamic_events()))
    assert all(keys[k] == (e.l_s, e.l_e) for k, e in zip(kidx[ta.dyn == 1].tolist(), tr.dynamic_events()))


def test_unknown_phase_message_follows_reference_order():
    F0, B0 = PhaseId.parse("F:0"), PhaseId.parse("B:0")
    evs = [MemoryRequestEvent(0, 512, 0, 2, F0, PhaseId.parse("B:7")), MemoryRequestEvent(1, 512, 1, 3, F0, B0)]
    ta = soa.from_events(evs, [PhaseSpan(F0, 0, 2), PhaseSpan(B0, 2, 10)])
    assert api._unknown_phase_message(ta) == "phase B:7 not in schedule"


def test_reuse_window_errors_are_host_side():
    from paper_2507_16274_b200.domain import LayerSpan

    with pytest.raises(PlanError, match="unknown layer"):
        api._windows([("a", "nope")], (LayerSpan("a", 0, 1),))
    with pytest.raises(PlanError, match="ends before"):
        api._windows([("a", "b")], (LayerSpan("a", 5, 6), LayerSpan("b", 1, 2)))


def test_plan_file_round_trip(tmp_path):
    b = PlanBundle(4096, 512, (PlanDecision(3, 0, 512, 0, 4), PlanDecision(9, 512, 1024, 1, 3)),
                   {("a", "b"): IntervalSet([Interval(2048, 4096)])})
    p = tmp_path / "plan.json"
    planio.write_plan(b, p)
    assert planio.read_plan(p) == b
    txt = p.read_text()
    assert txt.endswith("\n") and '"version": 1' in txt
    bad = PlanBundle(1024, 512, (PlanDecision(1, 768, 512, 0, 1),), {})
    planio.write_plan(bad, p)
    with pytest.raises(PlanError, match="out of pool"):
        planio.read_plan(p)
