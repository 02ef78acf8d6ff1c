"""The reference's own golden vectors and acceptance criteria, run through this
package's drop-in API on the GPU (pkg/tests/*.py of the reference, cited per test)."""

import json
import random

import numpy as np
import pytest

import paper_2507_16274_b200 as M
from paper_2507_16274_b200.domain import AllocationDecision, MemoryRequestEvent, PhaseId, PhaseSpan, Trace

pytestmark = pytest.mark.gpu
U = 512
MIB = 1 << 20


def make_trace(phases, events, layers=()):
    """conftest.make_trace (tests/conftest.py:6-31)."""
    spans = tuple(PhaseSpan(PhaseId.parse(t), s, e) for t, s, e in phases)
    evs = []
    for spec in events:
        eid, su, t_s, t_e, tag_s, tag_e, *rest = spec
        l_s, l_e = (rest + [None, None])[:2]
        evs.append(MemoryRequestEvent(eid, su * U, t_s, t_e, PhaseId.parse(tag_s), PhaseId.parse(tag_e),
                                      l_s is not None, l_s, l_e))
    return Trace(tuple(evs), spans, tuple(layers))


def sev(i, su, ts, te, a="F:0", b="B:0"):
    return MemoryRequestEvent(i, su * U, ts, te, PhaseId.parse(a), PhaseId.parse(b))


def conflict_pairs_oracle(decisions):
    """test_planner.py:293-302"""
    bad = []
    for i, a in enumerate(decisions):
        for b in decisions[i + 1:]:
            if a.t_s < b.t_e and b.t_s < a.t_e and a.addr < b.end_addr and b.addr < a.end_addr:
                bad.append((a, b))
    return bad


# ---------------------------------------------------------------- planner
def test_single_scoped_event():  # test_planner.py:273-281
    tr = make_trace([("F:0", 0, 1), ("B:0", 1, 2)], [(0, 8, 0, 1, "F:0", "B:0")])
    plan = M.synthesize_static_plan(tr)
    assert plan.pool_size == 8 * U == 4096
    assert len(plan.decisions) == 1 and plan.decisions[0].addr == 0
    assert M.peak_live_bytes(tr.events) / plan.pool_size == 1.0


def test_disjoint_same_size_share_one_layer():  # test_planner.py:284-290
    k = 5
    tr = make_trace([("F:0", 0, 2 * k)], [(i, 4, 2 * i, 2 * i + 1, "F:0", "F:0") for i in range(k)])
    plan = M.synthesize_static_plan(tr)
    assert plan.pool_size == 4 * U and len({d.addr for d in plan.decisions}) == 1


def test_touching_lifespans_do_not_share_a_layer():  # SURVEY App. A.1 (closed intervals)
    tr = make_trace([("F:0", 0, 9)], [(0, 4, 0, 5, "F:0", "F:0"), (1, 4, 5, 9, "F:0", "F:0")])
    assert M.synthesize_static_plan(tr).pool_size == 8 * U


def test_randomized_dense_valid_and_bounded():  # test_planner.py:305-316
    tr = M.synth_trace(M.SynthConfig.for_preset("dense", seed=9, num_layers=16, num_microbatches=10,
                                                transient_ratio=0.5))
    plan = M.synthesize_static_plan(tr)
    assert conflict_pairs_oracle(plan.decisions) == [] and M.validate_plan(plan) == []
    lb = M.peak_live_bytes(tr.static_events())
    assert lb <= plan.pool_size <= 1.10 * lb


def test_fusion_monotonicity_determinism_persistents():  # test_planner.py:319-343
    for preset in ("dense", "moe", "dense_vpp"):
        st = M.PlanStats()
        M.synthesize_static_plan(M.synth_trace(M.SynthConfig.for_preset(preset, seed=1)), stats=st)
        assert all(f > a for f, a in st.accepted_fusions)
    tr = M.synth_trace(M.SynthConfig.for_preset("dense_vpp", seed=3))
    a, b = M.synthesize_static_plan(tr), M.synthesize_static_plan(tr)
    assert a.pool_size == b.pool_size and [(d.id, d.addr) for d in a.decisions] == [(d.id, d.addr) for d in b.decisions]
    tr = M.synth_trace(M.SynthConfig.for_preset("dense", seed=0))
    plan = M.synthesize_static_plan(tr)
    persist = [d for d in plan.decisions if d.t_e >= tr.horizon]
    assert persist and max(d.end_addr for d in persist) == plan.persistent_size
    assert min(d.addr for d in plan.decisions if d.t_e < tr.horizon) >= plan.persistent_size


def test_ablations_do_not_break_validity():  # test_planner.py:346-354
    tr = M.synth_trace(M.SynthConfig.for_preset("moe_recompute", seed=2))
    for fusion in (True, False):
        for gap in (True, False):
            assert M.validate_plan(M.synthesize_static_plan(tr, fusion=fusion, gap_insert=gap)) == []
    assert M.synthesize_static_plan(tr, gap_insert=False).pool_size >= M.synthesize_static_plan(tr).pool_size


def test_validate_plan_examples():  # test_planner.py:371-402 + SURVEY §7 under-report case
    mk = lambda decs: M.StaticPlan(100 * U, U, tuple(decs), (), 0)  # noqa: E731
    assert M.validate_plan(mk([AllocationDecision(sev(0, 10, 0, 5), 0),
                               AllocationDecision(sev(1, 10, 3, 8), 10 * U)])) == []
    pairs = M.validate_plan(mk([AllocationDecision(sev(0, 10, 0, 5), 0), AllocationDecision(sev(1, 10, 3, 8), 0)]))
    assert len(pairs) == 1 and {pairs[0][0].id, pairs[0][1].id} == {0, 1}
    assert M.validate_plan(mk([AllocationDecision(sev(0, 10, 0, 5), 0), AllocationDecision(sev(1, 10, 0, 5), 10 * U),
                               AllocationDecision(sev(2, 10, 5, 9), 0)])) == []
    decs = [AllocationDecision(sev(0, 100, 0, 9), 0), AllocationDecision(sev(1, 10, 1, 9), 10 * U),
            AllocationDecision(sev(2, 10, 2, 9), 50 * U)]
    assert [(a.id, b.id) for a, b in M.validate_plan(mk(decs))] == [(0, 1)]


def test_plan_errors():
    tr = make_trace([("F:0", 0, 4)], [(0, 1, 0, 2, "F:0", "F:0")])
    bad = Trace((MemoryRequestEvent(7, 700, 0, 2, PhaseId.parse("F:0"), PhaseId.parse("F:0")),), tr.phase_schedule)
    with pytest.raises(M.PlanError, match="event 7: size 700 not aligned"):
        M.synthesize_static_plan(bad)
    unk = Trace((MemoryRequestEvent(1, 512, 0, 2, PhaseId.parse("F:0"), PhaseId.parse("B:9")),), tr.phase_schedule)
    with pytest.raises(M.TraceError, match="phase B:9 not in schedule"):
        M.synthesize_static_plan(unk)
    # times past the horizon (model.py:240-241) are rejected up front, and the
    # gap-insertion layer path must not index past the trace's timeline
    late = Trace((MemoryRequestEvent(1, 512, 0, 2, PhaseId.parse("F:0"), PhaseId.parse("F:0")),
                  MemoryRequestEvent(2, 512, 1, 9000, PhaseId.parse("F:0"), PhaseId.parse("F:0"))), tr.phase_schedule)
    with pytest.raises(M.TraceError, match="event 2: timestamps outside"):
        M.synthesize_static_plan(late)


# ---------------------------------------------------------------- reuse
def static_plan(specs, pool_u=100):  # test_reuse.py:28-38
    decs = tuple(AllocationDecision(sev(i, s, ts, te), a * U) for i, s, ts, te, a in specs)
    return M.StaticPlan(pool_u * U, U, decs, (), 0)


def sched(**spans):
    from paper_2507_16274_b200.domain import LayerSpan

    return tuple(LayerSpan(k, s, e) for k, (s, e) in spans.items())


def test_reusable_space_examples():  # test_reuse.py:74-100
    (lo, hi), space = M.compute_reusable_space(static_plan([(0, 100, 0, 10, 0)]), ("a", "b"), sched(a=(12, 14), b=(14, 15)))
    assert (lo, hi) == (12, 15) and space == M.IntervalSet.span(0, 100 * U)
    _, space = M.compute_reusable_space(static_plan([(0, 100, 0, 10, 0)]), ("a", "b"), sched(a=(5, 6), b=(7, 8)))
    assert space == M.IntervalSet.empty()
    plan = static_plan([(0, 40, 0, 10, 0), (1, 60, 20, 30, 40)])
    assert M.compute_reusable_space(plan, ("a", "b"), sched(a=(12, 15), b=(15, 18)))[1] == M.IntervalSet.span(0, 100 * U)
    assert M.compute_reusable_space(plan, ("a", "b"), sched(a=(8, 10), b=(20, 22)))[1] == M.IntervalSet.empty()
    with pytest.raises(M.PlanError, match="unknown layer"):
        M.compute_reusable_space(static_plan([(0, 10, 0, 5, 0)]), ("a", "nope"), sched(a=(0, 1)))


def test_reusable_space_brute_force_fuzz():  # test_reuse.py:103-135
    rng = random.Random(1)
    for _ in range(40):
        specs, addr = [], 0
        for i in range(rng.randint(1, 8)):
            size = rng.randint(1, 10)
            t_s = rng.randint(0, 30)
            specs.append((i, size, t_s, t_s + rng.randint(1, 15), addr))
            addr += size
        plan = static_plan(specs, pool_u=addr)
        t_lo = rng.randint(0, 30)
        t_hi = t_lo + rng.randint(1, 15)
        _, space = M.compute_reusable_space(plan, ("a", "b"), sched(a=(t_lo, t_lo + 1), b=(max(t_lo, t_hi - 1), t_hi)))
        free = []
        lo = min(d.addr for d in plan.decisions) // U
        hi = max(d.end_addr for d in plan.decisions) // U
        for unit in range(lo, hi):
            a = unit * U
            if not any(d.addr <= a < d.end_addr and d.t_s < t_hi and t_lo < d.t_e for d in plan.decisions):
                free.append(unit)
        assert space == M.IntervalSet(M.Interval(u * U, (u + 1) * U) for u in free)


def test_derive_reuse_map_keys_and_safety():  # test_reuse.py:166-190
    tr = M.synth_trace(M.SynthConfig.for_preset("moe", seed=5))
    plan, rmap = M.plan_trace(tr)
    assert set(rmap.entries) == set(M.group_dynamic(tr.dynamic_events()))
    for key, entry in rmap.entries.items():
        for d in plan.decisions:
            if d.t_s < entry.t_hi and entry.t_lo < d.t_e:
                for iv in entry.space:
                    assert iv.hi <= d.addr or d.end_addr <= iv.lo


# ---------------------------------------------------------------- replay + baseline
def test_self_simulation_dense():  # test_sim.py:21-30
    tr = M.synth_trace(M.SynthConfig.for_preset("dense", seed=0))
    plan, rmap = M.plan_trace(tr)
    rep, _ = M.simulate(tr, plan.to_bundle(rmap))
    assert rep.mismatch_count == 0 and rep.fallback_count == 0 and rep.reserved_peak == plan.pool_size
    assert rep.efficiency == pytest.approx(M.clique_lower_bound(tr) / plan.pool_size)


def test_replay_audit_and_safety():  # test_sim.py:122-167
    for preset in ("moe", "moe_recompute", "dense_vpp"):
        tr = M.synth_trace(M.SynthConfig.for_preset(preset, seed=2))
        plan, rmap = M.plan_trace(tr)
        _, log = M.simulate(tr, plan.to_bundle(rmap))
        live, bal = {}, 0
        for rec in log:
            if rec["kind"] == "alloc":
                span = (rec["space"], rec["addr"], rec["addr"] + rec["size"])
                for o in live.values():
                    if o[0] == span[0]:
                        assert not (span[1] < o[2] and o[1] < span[2])
                live[rec["id"]] = span
                bal += rec["size"]
            elif rec["kind"] == "free":
                live.pop(rec["id"])
                bal -= rec["size"]
        assert bal == 0 and not live
    tr = M.synth_trace(M.SynthConfig.for_preset("moe_recompute", seed=7))
    plan, rmap = M.plan_trace(tr)
    bundle = plan.to_bundle(rmap)
    _, log = M.simulate(tr, bundle)
    ev = {e.id: e for e in tr.events}
    pool_dyn = [r for r in log if r["kind"] == "alloc" and r["route"] == "reuse"]
    assert pool_dyn
    for r in pool_dyn:
        e = ev[r["id"]]
        for d in bundle.decisions:
            if d.t_s < e.t_e and e.t_s < d.t_e:
                assert r["addr"] + r["size"] <= d.addr or d.addr + d.size <= r["addr"]


def test_reuse_lowers_fallback_pressure_and_log_file(tmp_path):  # test_sim.py:170-218
    tr = M.synth_trace(M.SynthConfig.for_preset("moe_recompute", seed=1))
    plan, rmap = M.plan_trace(tr)
    b = plan.to_bundle(rmap)
    w, _ = M.simulate(tr, b)
    wo, _ = M.simulate(tr, b, reuse=False)
    assert w.fallback_bytes_peak <= wo.fallback_bytes_peak and w.reserved_peak <= wo.reserved_peak
    assert w.reuse_hits > 0 and wo.reuse_hits == 0
    tr = M.synth_trace(M.SynthConfig.for_preset("dense", seed=0))
    plan, rmap = M.plan_trace(tr)
    out = tmp_path / "log.jsonl"
    M.simulate(tr, plan.to_bundle(rmap), log_path=out)
    lines = out.read_text().splitlines()
    assert lines[0] == '{"kind":"init","pool_size":%d}' % plan.pool_size
    assert len(lines) == 1 + 2 * len(tr.events)
    assert json.loads(lines[1])["kind"] == "alloc"


def test_baseline_examples():  # test_baseline.py:15-46
    A, B = 4 * MIB // U, 2 * MIB // U
    rep = M.run_baseline(make_trace([("F:0", 0, 10)], [(i, A, 2 * i, 2 * i + 1, "F:0", "F:0") for i in range(5)]))
    assert (rep.reserved_peak, rep.allocated_peak, rep.efficiency) == (4 * MIB, 4 * MIB, 1.0)
    rep = M.run_baseline(make_trace([("F:0", 0, 8)], [(1, A, 0, 2, "F:0", "F:0"), (2, B, 1, 5, "F:0", "F:0"),
                                                      (3, B, 3, 6, "F:0", "F:0"), (4, A, 4, 7, "F:0", "F:0")]))
    assert (rep.allocated_peak, rep.reserved_peak) == (8 * MIB, 10 * MIB)
    assert rep.efficiency == pytest.approx(0.8) and rep.fragmentation == pytest.approx(0.2)


def test_duplicate_ids_surface_as_simulation_error():  # test_sim.py:107-119
    F = PhaseId.parse("F:0")
    tr = Trace((MemoryRequestEvent(0, U, 0, 2, F, F), MemoryRequestEvent(0, U, 1, 3, F, F)), (PhaseSpan(F, 0, 4),))
    with pytest.raises(M.SimulationError, match="already live|double free|unknown"):
        M.simulate(tr, M.PlanBundle(0, U, (), {}))


# ---------------------------------------------------------------- acceptance (test_acceptance.py)
def fuzz_config(seed):  # test_acceptance.py:28-36
    return M.SynthConfig.for_preset(M.PRESETS[seed % 6], seed=seed, num_layers=4 + seed % 9,
                                    num_microbatches=1 + seed % 4, transient_ratio=0.2 + (seed % 5) * 0.2)


def test_criteria_1_and_7_fuzz_validity_and_fusion_monotonicity():
    accepted = 0
    for seed in range(200):
        tr = M.synth_trace(fuzz_config(seed))
        st = M.PlanStats()
        plan, _ = M.plan_trace(tr, stats=st)
        assert M.validate_plan(plan) == []
        assert all(f > a for f, a in st.accepted_fusions)
        accepted += len(st.accepted_fusions)
    assert accepted > 0


def test_criteria_3_4_dense_efficiency_and_baseline_contrast():
    effs = []
    for preset in ("dense", "dense_recompute", "dense_vpp"):
        for seed in range(5):
            tr = M.synth_trace(M.SynthConfig.for_preset(preset, seed=seed))
            plan, _ = M.plan_trace(tr)
            effs.append(M.clique_lower_bound(tr) / plan.pool_size)
    assert min(effs) >= 0.95
    fp, fb = [], []
    for preset in ("dense_recompute", "dense_vpp"):
        for seed in range(5):
            tr = M.synth_trace(M.SynthConfig.for_preset(preset, seed=seed))
            plan, rmap = M.plan_trace(tr)
            p, _ = M.simulate(tr, plan.to_bundle(rmap))
            b = M.run_baseline(tr)
            assert b.efficiency < p.efficiency
            fp.append(p.fragmentation)
            fb.append(b.fragmentation)
    assert sum(fp) / len(fp) <= 0.5 * sum(fb) / len(fb)


def test_criteria_5_6_dynamic_reuse_safety_and_benefit():
    placements = 0
    for seed in range(100):
        preset = "moe" if seed % 2 == 0 else "moe_recompute"
        tr = M.synth_trace(M.SynthConfig.for_preset(preset, seed=seed, num_layers=4 + seed % 7,
                                                    num_microbatches=1 + seed % 3))
        plan, rmap = M.plan_trace(tr)
        b = plan.to_bundle(rmap)
        _, log = M.simulate(tr, b)
        ev = {e.id: e for e in tr.events}
        for r in log:
            if r["kind"] == "alloc" and r["route"] == "reuse":
                placements += 1
                e = ev[r["id"]]
                for d in b.decisions:
                    if d.t_s < e.t_e and e.t_s < d.t_e:
                        assert not (r["addr"] < d.addr + d.size and d.addr < r["addr"] + r["size"])
    assert placements > 0
    wins = 0
    for seed in range(10):
        tr = M.synth_trace(M.SynthConfig.for_preset("moe_recompute", seed=seed))
        plan, rmap = M.plan_trace(tr)
        b = plan.to_bundle(rmap)
        w, _ = M.simulate(tr, b)
        wo, _ = M.simulate(tr, b, reuse=False)
        wins += w.fallback_bytes_peak < wo.fallback_bytes_peak and w.reserved_peak < wo.reserved_peak
    assert wins >= 8


def test_criterion_8_scale_and_10_self_simulation_closure():
    import time

    tr = M.synth_trace(M.SynthConfig.for_preset("dense_recompute", seed=0, num_layers=128, num_microbatches=160,
                                                transient_ratio=1.0))
    t0 = time.monotonic()
    plan, _ = M.plan_trace(tr)
    assert len(tr.events) >= 100_000 and time.monotonic() - t0 < 120.0
    assert plan.pool_size >= M.peak_live_bytes(tr.static_events())
    for preset in M.PRESETS:
        tr = M.synth_trace(M.SynthConfig.for_preset(preset, seed=0))
        plan, rmap = M.plan_trace(tr)
        rep, _ = M.simulate(tr, plan.to_bundle(rmap))
        assert rep.mismatch_count == 0 and (rep.fallback_count == 0 or preset.startswith("moe"))
