"""The reference planner's sub-operations through libstw (stw_group_events,
stw_local_plans, stw_weighted_tmp, stw_fuse_plans, stw_build_layers,
stw_metrics), imported through the reference's module paths.

Known answers are the reference's own pins (pkg/tests/test_planner.py:61-181,
:225-266; test_acceptance.py:60-84; test_sim.py:181-200), restated here;
randomized cases are checked against oracle/subops.py and CPython's own float
arithmetic (bit-exact: `==`, never approx)."""

import random

import pytest

from oracle import subops as O
from paper_2507_16274_b200.domain import AllocationDecision, MemoryRequestEvent, PhaseId, PlanError
from paper_2507_16274_b200.planner import (
    HomoPhaseGroup,
    LocalPlan,
    _Item,
    _plan_from_decisions,
    build_layers_for_size,
    compute_tmp,
    fuse_plans,
    group_by_phase,
    pack_group,
    pack_groups,
    try_fuse,
    weighted_tmp_average,
)

pytestmark = pytest.mark.gpu
U = 512
P = PhaseId.parse


def ev(i, su, ts, te, a="F:0", b="B:0"):
    return MemoryRequestEvent(i, su * U, ts, te, P(a), P(b))


def plan_of(specs, key=("F:0", "B:0")):
    """specs: (id, size_u, t_s, t_e, addr_u)"""
    return _plan_from_decisions((P(key[0]), P(key[1])),
                                [AllocationDecision(ev(i, s, a, b, *key), d * U) for i, s, a, b, d in specs])


def rects(plan):
    return [(d.id, d.size, d.t_s, d.t_e, d.addr) for d in plan.decisions]


# ---------------------------------------------------------------------------
# group_by_phase


def test_group_by_phase_partition():
    events = [ev(i, 1, i, i + 10, "F:0", "B:0") for i in range(3)] + [ev(3 + i, 1, i, i + 10, "F:1", "B:1")
                                                                      for i in range(2)]
    groups = group_by_phase(events)
    assert [len(g.members) for g in groups] == [3, 2]
    assert [g.key[0].tag() for g in groups] == ["F:0", "F:1"]
    for g in groups:
        assert list(g.members) == sorted(g.members, key=lambda e: (e.t_s, e.id))


def test_group_by_phase_empty_and_single_group():
    assert group_by_phase([]) == []
    groups = group_by_phase([ev(i, 1, i, 100, "init", "opt") for i in range(4)])
    assert len(groups) == 1 and groups[0].key == (P("init"), P("opt"))


def test_group_by_phase_rejects_dynamic():
    d = MemoryRequestEvent(0, U, 0, 1, P("F:0"), P("F:0"), True, "a", "a")
    with pytest.raises(PlanError, match="dynamic"):
        group_by_phase([d])


def test_group_by_phase_random_vs_oracle():
    rng = random.Random(7)
    tags = ["init", "F:0", "F:1", "B:1", "B:0", "F:2.1", "B:2.1", "opt"]
    for _ in range(20):
        evs = []
        for i in rng.sample(range(1000), rng.randint(1, 60)):
            a, b = sorted(rng.sample(range(len(tags)), 2))
            t = rng.randint(0, 50)
            evs.append(ev(i, rng.randint(1, 9), t, t + rng.randint(1, 9), tags[a], tags[b]))
        got = [(g.key, [e.id for e in g.members]) for g in group_by_phase(evs)]
        want = [(k, [e[0] for e in m]) for k, m in O.group_keys([(e.id, e.t_s, e.p_s, e.p_e) for e in evs])]
        assert got == want


# ---------------------------------------------------------------------------
# packing and TMP (bit-exact against Python int / int)


def test_pack_group_prefix_sums():
    g = HomoPhaseGroup((P("F:0"), P("B:0")), (ev(0, 60, 0, 10), ev(1, 40, 0, 4)))
    plan = pack_group(g)
    assert [d.addr for d in plan.decisions] == [0, 60 * U]
    assert plan.height == 100 * U and (plan.t_s, plan.t_e) == (0, 10)
    assert plan.tmp == (600 + 160) * U / (100 * U * 10)


def test_tmp_single_and_time_shared():
    assert compute_tmp(plan_of([(0, 10, 0, 5, 0)])) == 1.0
    p = plan_of([(0, 10, 0, 2, 0), (1, 10, 3, 5, 0)])
    assert p.height == 10 * U and compute_tmp(p) == 40 / 50


def test_tmp_zero_duration_errors():
    p = LocalPlan((P("F:0"), P("F:0")), (AllocationDecision(ev(0, 1, 5, 6), 0),), height=U, t_s=5, t_e=5, tmp=0.0)
    with pytest.raises(PlanError, match="degenerate lifespan"):
        compute_tmp(p)


def test_pack_empty_group_errors():
    with pytest.raises(PlanError, match="empty group"):
        pack_group(HomoPhaseGroup((P("F:0"), P("B:0")), ()))


def test_pack_groups_random_bit_exact():
    rng = random.Random(3)
    groups = []
    for g in range(64):
        n = rng.randint(1, 40)
        groups.append(HomoPhaseGroup((P("F:0"), P("B:0")), tuple(
            ev(1000 * g + i, rng.randint(1, 1 << 20), t := rng.randint(0, 1 << 20), t + rng.randint(1, 1 << 18))
            for i in range(n))))
    for g, p in zip(groups, pack_groups(groups)):
        addrs, a = [], 0
        for m in g.members:
            addrs.append(a)
            a += m.size
        assert [d.addr for d in p.decisions] == addrs
        assert (p.height, p.t_s, p.t_e, p.tmp) == O.plan_box(rects(p))


# ---------------------------------------------------------------------------
# fusion


def test_try_fuse_accepts_nested_smaller():
    larger = plan_of([(0, 60, 0, 10, 0), (1, 40, 0, 4, 60)])
    smaller = plan_of([(2, 40, 5, 9, 0)], key=("F:0", "F:0"))
    assert larger.tmp == 0.76 and smaller.tmp == 1.0
    fused = try_fuse(larger, smaller)
    assert fused is not None and fused.height == 100 * U
    assert {d.id: d.addr for d in fused.decisions}[2] == 60 * U
    assert fused.tmp == (600 + 160 + 160) / 1000
    avg = weighted_tmp_average([larger, smaller])
    assert avg == O.weighted([(larger.tmp, larger.space_time), (smaller.tmp, smaller.space_time)])
    assert fused.tmp > avg


def test_fuse_stacks_on_top_when_everything_overlaps():
    larger = plan_of([(0, 50, 0, 10, 0), (1, 50, 0, 10, 50)])
    smaller = plan_of([(2, 10, 0, 10, 0)], key=("F:0", "F:0"))
    fused = fuse_plans(larger, smaller)
    assert {d.id: d.addr for d in fused.decisions}[2] == 100 * U
    assert fused.tmp == 1.0 and weighted_tmp_average([larger, smaller]) == 1.0
    assert try_fuse(larger, smaller) is None  # not strictly better


def test_try_fuse_rejects_strictly_worse():
    larger = plan_of([(0, 60, 0, 10, 0), (1, 40, 2, 8, 60)])
    smaller = plan_of([(2, 30, 1, 9, 0)], key=("F:0", "F:0"))
    fused = fuse_plans(larger, smaller)
    assert fused.height == 130 * U and fused.tmp == 1080 / 1300
    assert weighted_tmp_average([larger, smaller]) == 1080 / 1240
    assert try_fuse(larger, smaller) is None


def test_try_fuse_empty_plan_passthrough():
    larger = plan_of([(0, 10, 0, 5, 0)])
    empty = LocalPlan(larger.key, (), 0, 0, 0, 0.0)
    assert try_fuse(larger, empty) is larger and fuse_plans(empty, larger) is larger


def test_fused_key_rule():
    larger = plan_of([(0, 60, 2, 10, 0)], key=("F:1", "B:1"))
    smaller = plan_of([(1, 10, 0, 4, 0)], key=("F:0", "B:0"))
    fused = fuse_plans(larger, smaller)
    assert fused.key == (P("F:0"), P("B:1"))  # planner.py:165-168


def test_fusion_random_vs_oracle():
    """Placement, numerator invariance and acceptance <=> space-time shrink
    (test_planner.py:184-214), placements against the cursor-walk oracle."""
    rng = random.Random(0)
    for _ in range(60):
        big = pack_group(HomoPhaseGroup((P("F:0"), P("B:0")), tuple(
            ev(i, rng.randint(1, 20), s := rng.randint(0, 10), s + rng.randint(1, 10)) for i in range(rng.randint(1, 6)))))
        small = pack_group(HomoPhaseGroup((P("F:0"), P("F:0")), tuple(
            ev(100 + i, rng.randint(1, 10), s := rng.randint(0, 10), s + rng.randint(1, 8), "F:0", "F:0")
            for i in range(rng.randint(1, 5)))))
        if small.height > big.height:
            big, small = small, big
        fused = fuse_plans(big, small)
        want, order = O.fuse(rects(big), rects(small))
        assert [d.id for d in fused.decisions[len(big.decisions):]] == order
        assert {d.id: d.addr for d in fused.decisions[len(big.decisions):]} == want
        assert (fused.height, fused.t_s, fused.t_e, fused.tmp) == O.plan_box(rects(fused))
        accepted = try_fuse(big, small)
        avg = O.weighted([(big.tmp, big.space_time), (small.tmp, small.space_time)])
        assert (accepted is not None) == (fused.tmp > avg)
        assert (accepted is not None) == (fused.space_time < big.space_time + small.space_time)


def test_weighted_average_many_plans_cpython_semantics():
    rng = random.Random(11)
    for _ in range(20):
        plans = [plan_of([(k, rng.randint(1, 99), s := rng.randint(0, 50), s + rng.randint(1, 40), 0)])
                 for k in range(rng.randint(2, 9))]
        plans = [LocalPlan(p.key, p.decisions, p.height, p.t_s, p.t_e, rng.random()) for p in plans]
        assert weighted_tmp_average(plans) == sum(p.tmp * p.space_time for p in plans) / sum(
            p.space_time for p in plans)


# ---------------------------------------------------------------------------
# memory layers (Alg. 1)


def items_of(spans, size_u=4):
    return [_Item(size_u * U, s, e, i, ev(i, size_u, int(s), int(e) + 1)) for i, (s, e) in enumerate(spans)]


def test_build_layers_spec_example():
    layers = build_layers_for_size(items_of([(0, 2), (1, 3), (2.5, 4)]))
    assert len(layers) == 2
    assert [s[0] for s in layers[0].slots] == [0, 2.5]  # C joined the layer that ended at 2
    assert layers[0].end == 4 and layers[0].size == 4 * U


def test_build_layers_disjoint_and_all_overlapping():
    assert len(build_layers_for_size(items_of([(0, 1), (2, 3), (4, 5), (6, 7)]))) == 1
    assert len(build_layers_for_size(items_of([(0, 10), (1, 10), (2, 10), (3, 10)]))) == 4


def test_build_layers_touching_is_closed():
    assert len(build_layers_for_size(items_of([(0, 5), (5, 9)]))) == 2


def test_build_layers_fuzz_vs_oracle():
    rng = random.Random(5)
    for _ in range(200):
        spans = []
        for _ in range(rng.randint(1, 50)):
            s = rng.randint(0, 60)
            spans.append((s, s + rng.randint(1, 25)))
        items = items_of(spans)
        layers = build_layers_for_size(items)
        assert len(layers) == O.closed_overlap(spans)
        want, nl = O.alg1([(i.t_s, i.t_e, i.tie) for i in items])
        got = {}
        for li, layer in enumerate(layers):
            for _, _, k in layer.slots:
                got[k.value.id] = li
        assert [got[i] for i in range(len(items))] == want and nl == len(layers)


def test_acceptance_criterion_2_layer_count_optimality():
    """test_acceptance.py:60-84: 1000 random instances, layer count == the
    closed-interval clique number."""
    rng = random.Random(2024)
    for i in range(1000):
        spans = []
        for _ in range(rng.randint(1, 50)):
            s = rng.randint(0, 80)
            spans.append((s, s + rng.randint(1, 30)))
        layers = build_layers_for_size([_Item(512, s, e, j, None) for j, (s, e) in enumerate(spans)])
        assert len(layers) == O.closed_overlap(spans), i


def test_memory_layer_fits_gap_and_insert():
    from paper_2507_16274_b200.planner import MemoryLayer

    layer = MemoryLayer(size=8 * U)
    layer.insert(10, 20, "a")
    layer.insert(0, 4, "b")
    assert [s[:2] for s in layer.slots] == [(0, 4), (10, 20)] and layer.end == 20
    assert layer.fits_gap(5, 9) and not layer.fits_gap(4, 9) and not layer.fits_gap(5, 10)
    assert layer.slots[1][2].value == "a"


# ---------------------------------------------------------------------------
# compute_metrics


def test_compute_metrics_known_answers():
    from paper_2507_16274_b200.sim import compute_metrics

    exact = [{"kind": "init", "pool_size": 100},
             {"kind": "alloc", "t": 0, "id": 0, "size": 100, "space": "pool", "addr": 0, "route": "planned"},
             {"kind": "free", "t": 1, "id": 0, "size": 100, "space": "pool", "addr": 0}]
    rep = compute_metrics(exact)
    assert rep.efficiency == 1.0 and rep.fragmentation == 0.0
    rep = compute_metrics(exact[:1] + [dict(exact[1], size=90)])
    assert (rep.allocated_peak, rep.reserved_peak, rep.fragmentation) == (90, 100, 1.0 - 90 / 100)


@pytest.mark.parametrize("preset,seed", [("moe", 2), ("moe_recompute", 1), ("dense_vpp", 0)])
def test_compute_metrics_of_replay_logs(preset, seed):
    import paper_2507_16274_b200 as M
    from paper_2507_16274_b200 import tracegen
    from paper_2507_16274_b200.sim import compute_metrics

    tr = M.synth_trace(tracegen.SynthConfig.for_preset(preset, seed=seed))
    plan, rmap = M.plan_trace(tr)
    for reuse in (True, False):
        rep, log = M.simulate(tr, plan.to_bundle(rmap), reuse=reuse)
        assert compute_metrics(log) == rep  # columns straight from the device log
        dicts = list(log)
        assert compute_metrics(dicts) == rep == M.SimReport(**O.metrics(dicts))
    base = M.run_baseline(tr)
    assert base.reserved_peak >= M.clique_lower_bound(tr)
