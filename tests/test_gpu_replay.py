"""Reuse map (K8), replay scorer (K9) and caching-allocator baseline (K10):
libstw vs the C oracle, bit-exact (reports, every log record, every interval)."""

import numpy as np
import pytest

from paper_2507_16274_b200 import api, tracegen
from oracle import oracle as O

pytestmark = pytest.mark.gpu

KIND = {0: "init", 1: "reserve", 2: "alloc", 3: "free"}


def fuzz_cfg(seed):
    preset = tracegen.PRESETS[seed % 6]
    return tracegen.SynthConfig.for_preset(preset, seed=seed, num_layers=4 + seed % 9,
                                          num_microbatches=1 + seed % 4, transient_ratio=0.2 + (seed % 5) * 0.2)


def oracle_inputs(ta, bundle):
    names, kidx = ta.dynamic_keys()
    bkeys = list(bundle.reuse)
    pos = {k: i for i, k in enumerate(bkeys)}
    key = np.array([pos.get(names[k], -1) if k >= 0 else -1 for k in kidx], np.int32)
    off, lo, hi = [0], [], []
    for k in bkeys:
        for iv in bundle.reuse[k]:
            lo.append(iv.lo)
            hi.append(iv.hi)
        off.append(len(lo))
    c = bundle._cols
    return key, (c.id, c.addr, c.size, c.t_s, c.t_e), off, lo, hi


def oracle_log_dicts(lg, ta):
    evkey = {int(ta.id[i]): [ta.layer_names[ta.ls[i]], ta.layer_names[ta.le[i]]] for i in np.nonzero(ta.dyn)[0]}
    routes = ("planned", "reuse", "fallback", "mismatch", "online")
    out = []
    for k in range(len(lg["kind"])):
        kind = KIND[int(lg["kind"][k])]
        if kind == "init":
            out.append({"kind": "init", "pool_size": int(lg["size"][k])})
        elif kind == "reserve":
            out.append({"kind": "reserve", "t": int(lg["t"][k]), "bytes": int(lg["size"][k])})
        else:
            r = {"kind": kind, "t": int(lg["t"][k]), "id": int(lg["id"][k]), "size": int(lg["size"][k]),
                 "space": "pool" if lg["space"][k] == 0 else "cache", "addr": int(lg["addr"][k])}
            if kind == "alloc":
                r["route"] = routes[int(lg["route"][k])]
                if r["id"] in evkey:
                    r["key"] = evkey[r["id"]]
            out.append(r)
    return out


def check_trace(ta, reuse_flags=(True, False)):
    tr = api.Trace.from_arrays(ta) if hasattr(api, "Trace") else None
    from paper_2507_16274_b200.domain import Trace

    tr = Trace.from_arrays(ta)
    plan, rmap = api.plan_trace(tr)
    cols = plan.columns()
    # K8 vs oracle
    keys = list(rmap.entries)
    if keys:
        t_lo = [rmap.entries[k].t_lo for k in keys]
        t_hi = [rmap.entries[k].t_hi for k in keys]
        off, lo, hi = O.reuse(cols.addr, cols.size, cols.t_s, cols.t_e, t_lo, t_hi)
        for i, k in enumerate(keys):
            got = [(iv.lo, iv.hi) for iv in rmap.entries[k].space]
            assert got == list(zip(lo[off[i]:off[i + 1]].tolist(), hi[off[i]:off[i + 1]].tolist())), k
    bundle = plan.to_bundle(rmap)
    key, dcols, off, lo, hi = oracle_inputs(ta, bundle)
    for reuse in reuse_flags:
        rep, log = api.simulate(tr, bundle, reuse=reuse)
        o = O.simulate(ta, key, bundle.pool_size, bundle.alignment, *dcols, off, lo, hi, reuse)
        assert o.rc == 0, o.err
        assert rep.to_dict() == o.report
        assert list(log) == oracle_log_dicts(o.log, ta)
    b = api.run_baseline(tr)
    ob = O.baseline(ta)
    assert b.to_dict() == ob.report
    return rep


def test_replay_fuzz():
    for s in range(48):
        check_trace(tracegen.synth_arrays(fuzz_cfg(s)))


@pytest.mark.parametrize("name", ["c1_llama2_7b_1f1b", "c3_mixtral_moe", "c3b_mixtral_moe_rcp"])
def test_replay_configs(name):
    check_trace(tracegen.synth_arrays(tracegen.config(name)), (True,))


def test_replay_c2():
    check_trace(tracegen.synth_arrays(tracegen.config("c2_llama2_7b_vpp_rcp")), (True,))


def test_replay_mismatch_and_occupied():
    from paper_2507_16274_b200.domain import MemoryRequestEvent, PhaseId, PhaseSpan, SimulationError, Trace
    from paper_2507_16274_b200.plan_types import PlanBundle, PlanDecision

    U = 512
    F, B = PhaseId.parse("F:0"), PhaseId.parse("B:0")
    sched = (PhaseSpan(F, 0, 3), PhaseSpan(B, 3, 6))
    base = Trace((MemoryRequestEvent(0, 8 * U, 0, 4, F, B), MemoryRequestEvent(1, 4 * U, 1, 3, F, F)), sched)
    plan, rmap = api.plan_trace(base)
    injected = Trace(base.events + (MemoryRequestEvent(2, 16 * U, 2, 5, F, B),), sched)
    rep, log = api.simulate(injected, plan.to_bundle(rmap))  # test_sim.py:33-52
    assert rep.mismatch_count == 1 and rep.fallback_count == 1
    routes = {r["id"]: r["route"] for r in log if r["kind"] == "alloc"}
    assert routes == {0: "planned", 1: "planned", 2: "mismatch"}
    tr = Trace((MemoryRequestEvent(0, 8 * U, 0, 2, F, B), MemoryRequestEvent(1, 8 * U, 1, 3, F, B)),
               (PhaseSpan(F, 0, 2), PhaseSpan(B, 2, 4)))
    corrupt = PlanBundle(16 * U, U, (PlanDecision(0, 0, 8 * U, 0, 2), PlanDecision(1, 0, 8 * U, 1, 3)), {})
    with pytest.raises(SimulationError, match="occupied"):  # test_sim.py:92-104
        api.simulate(tr, corrupt)


def test_replay_fast_path_conflicts_fuzz():
    """Static-only traces take the parallel replay (K7 overlap test + prefix sums);
    corrupted plans must fall back and raise exactly like the oracle's sequential replay."""
    from paper_2507_16274_b200.domain import SimulationError, Trace
    from paper_2507_16274_b200.plan_types import PlanBundle, PlanDecision

    rng = np.random.default_rng(11)
    for s in range(24):
        ta = tracegen.synth_arrays(tracegen.c4_config(s))
        tr = Trace.from_arrays(ta)
        plan, rmap = api.plan_trace(tr)
        c = plan.columns()
        addr = c.addr.copy()
        if s % 3:  # move a few decisions onto other decisions' addresses (mostly conflicts)
            for _ in range(1 + s % 4):
                i, j = rng.integers(0, addr.size, 2)
                addr[i] = min(addr[j], plan.pool_size - int(c.size[i]))
        decs = tuple(PlanDecision(int(a), int(b), int(z), int(x), int(y))
                     for a, b, z, x, y in zip(c.id, addr, c.size, c.t_s, c.t_e))
        bundle = PlanBundle(plan.pool_size, plan.alignment, decs, {})
        key, dcols, off, lo, hi = oracle_inputs(ta, plan.to_bundle(rmap))
        o = O.simulate(ta, key, bundle.pool_size, bundle.alignment, dcols[0], addr, *dcols[2:], [0], [], [], True)
        if o.rc == 0:
            rep, log = api.simulate(tr, bundle)
            assert rep.to_dict() == o.report
            assert list(log) == oracle_log_dicts(o.log, ta)
        else:
            with pytest.raises(SimulationError) as ei:
                api.simulate(tr, bundle)
            assert str(o.err_id) in str(ei.value), (str(ei.value), o.err)


@pytest.mark.parametrize("general", [False, True])
def test_replay_fuzz_both_warps(general, monkeypatch):
    """The register-resident warp (replay_reg.cu) and the general warp
    (k_replay, forced by STW_REPLAY_GENERAL) give the oracle's exact reports and logs."""
    if general:
        monkeypatch.setenv("STW_REPLAY_GENERAL", "1")
    for s in range(48, 72):
        check_trace(tracegen.synth_arrays(fuzz_cfg(s)))


@pytest.mark.parametrize("k", [100, 200, 300, 600])
def test_replay_register_capacity(k):
    """k live requests of 3 MiB leave k cache segments with a 1 MiB free tail
    each: > 128 blocks outgrow 4 rows per lane, > 512 the register warp entirely
    (the call falls back to k_replay). Every size gives the oracle's report."""
    from paper_2507_16274_b200.domain import MemoryRequestEvent, PhaseId, PhaseSpan, Trace

    MIB = 1 << 20
    F, B = PhaseId.parse("F:0"), PhaseId.parse("B:0")
    sched = (PhaseSpan(F, 0, k), PhaseSpan(B, k, 2 * k + 1))
    evs = tuple(MemoryRequestEvent(i, 3 * MIB + 512 * (i % 3), i, k + 1 + i, F, B) for i in range(k))
    tr = Trace(evs, sched)
    b = api.run_baseline(tr)
    assert b.to_dict() == O.baseline(api._arrays_of(tr)).report


def test_replay_offchain_adversarial_spaces(monkeypatch, capfd):
    """Reuse spaces that overlap planned rectangles (the whole pool, or random
    windows of it) break the off-chain conditions: the call must notice and
    replay the full chain, matching the oracle (reports, logs, or the exact
    SimulationError). Unmodified bundles take the short chain."""
    from paper_2507_16274_b200.domain import SimulationError, Trace
    from paper_2507_16274_b200.ivset import Interval, IntervalSet
    from paper_2507_16274_b200.plan_types import PlanBundle

    monkeypatch.setenv("STW_REPLAY_STATS", "1")
    rng = np.random.default_rng(3)
    seen = {"off-planned": 0, "full": 0}
    for s in range(4, 40, 6):  # MoE presets (dynamic requests)
        ta = tracegen.synth_arrays(fuzz_cfg(s))
        tr = Trace.from_arrays(ta)
        plan, rmap = api.plan_trace(tr)
        good = plan.to_bundle(rmap)
        variants = [good]
        P, U = good.pool_size, good.alignment

        def bundle_with(spaces):
            nb = PlanBundle(P, U, good.decisions, spaces)
            object.__setattr__(nb, "_cols", good._cols)
            return nb

        whole = {k: IntervalSet([Interval(0, P)]) for k in good.reuse}
        variants.append(bundle_with(whole))
        rnd = {}
        for k in good.reuse:
            a = int(rng.integers(0, P // U)) * U
            b = min(P, a + int(rng.integers(1, 64)) * U * 256)
            rnd[k] = IntervalSet([Interval(a, b)])
        variants.append(bundle_with(rnd))
        for bundle in variants:
            key, dcols, off, lo, hi = oracle_inputs(ta, bundle)
            o = O.simulate(ta, key, bundle.pool_size, bundle.alignment, *dcols, off, lo, hi, True)
            capfd.readouterr()
            if o.rc == 0:
                rep, log = api.simulate(tr, bundle)
                assert rep.to_dict() == o.report, s
                assert list(log) == oracle_log_dicts(o.log, ta), s
            else:
                with pytest.raises(SimulationError) as ei:
                    api.simulate(tr, bundle)
                assert str(o.err_id) in str(ei.value), (str(ei.value), o.err)
            err = capfd.readouterr().err
            for k in seen:
                seen[k] += f"{k} chain" in err
    assert seen["off-planned"] > 0 and seen["full"] > 0, seen


def test_replay_shuffled_listing_takes_the_general_id_path():
    """Replay preprocessing skips the id sorts when ids increase along the
    listing (the usual trace); a shuffled listing takes the sorting path.
    Both match the oracle (reports and every log record)."""
    import dataclasses

    rng = np.random.default_rng(17)
    for s in (4, 5, 10, 11):
        ta = tracegen.synth_arrays(fuzz_cfg(s))
        p = rng.permutation(len(ta))
        sh = dataclasses.replace(ta, **{k: getattr(ta, k)[p] for k in
                                        ("id", "size", "t_s", "t_e", "ps", "pe", "dyn", "ls", "le")})
        check_trace(ta, (True,))
        check_trace(sh, (True,))
