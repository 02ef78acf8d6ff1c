"""Full-size parity on the device against the reference's own outputs
(tests/golden/anchors.json, made by running the reference):
plan file sha256, pool, PlanStats, replay report + log digest, baseline
report for c1/c2/c3/c3b/c5, and the c4 digest over 4096 traces x 4 candidates."""

import hashlib

import numpy as np
import pytest

import paper_2507_16274_b200 as M
from paper_2507_16274_b200 import api, planio, tracegen
from paper_2507_16274_b200.batching import HostBatch

from _util import anchors, fuzz_fixtures, log_digest, trace_digest

pytestmark = pytest.mark.gpu
STATS = ("events", "persistent", "phase_groups", "local_plans", "residual_events", "fusion_attempts",
         "fusion_accepted", "gap_insertions", "layers", "pool_size", "static_peak")


def run_config(name):
    a = anchors()[name]
    ta = tracegen.synth_arrays(tracegen.config(name))
    assert trace_digest(ta) == a["trace_digest"]
    tr = M.Trace.from_arrays(ta)
    st = M.PlanStats()
    plan, rmap = M.plan_trace(tr, stats=st)
    got = st.to_dict()
    for k in STATS:
        assert got[k] == a["stats"][k], k
    assert [list(x) for x in st.accepted_fusions] == a["accepted_fusions"]
    bundle = plan.to_bundle(rmap)
    sha = hashlib.sha256(planio.dumps_plan(bundle).encode()).hexdigest()[:16]
    assert sha == a["write_plan_sha16"]
    rep, log = M.simulate(tr, bundle)
    assert rep.to_dict() == a["sim"]
    assert log_digest(log) == a["sim_log_digest"]
    assert M.run_baseline(tr).to_dict() == a["baseline"]
    assert M.clique_lower_bound(tr) == a["clique_lower_bound"]


@pytest.mark.parametrize("name", ["c1_llama2_7b_1f1b", "c2_llama2_7b_vpp_rcp", "c3_mixtral_moe", "c3b_mixtral_moe_rcp"])
def test_app_b_config(name):
    run_config(name)


@pytest.mark.slow
def test_app_b_c5():
    run_config("c5_llama3_70b")


def test_c4_digest_full_sweep():
    """SURVEY App. B c4 recipe, all 16,384 plans from one batched device call."""
    a = anchors()["c4"]
    tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(4096)]
    hb = HostBatch(tas)
    bp = api.plan_batch(hb, tracegen.C4_CANDIDATES, select_best=True, detail=False)
    assert bp.rc.max() == 0
    lines = []
    total_best = 0
    for t, ta in enumerate(tas):
        s0, s1 = int(hb.ev_off[t]), int(hb.ev_off[t + 1])
        order = bp.order[s0:s1]
        order = order[ta.dyn[order] == 0]
        ids = ta.id[order].tolist()
        parts = []
        for c in range(4):
            addr = bp.addr[c, s0:s1][order].tolist()
            h8 = hashlib.sha256(",".join(f"{i}:{x}" for i, x in zip(ids, addr)).encode()).hexdigest()[:8]
            parts.append(f"{int(bp.stats[t * 4 + c, 9])}:{h8}")
        best = int(bp.best_cand[t])
        total_best += int(bp.best_pool[t])
        lines.append(f"{t}|{len(ids)}|{best}|" + "|".join(parts) + "\n")
    assert [ln.strip() for ln in lines[:8]] == a["lines_sha_first8"]
    assert hashlib.sha256("".join(lines).encode()).hexdigest()[:16] == a["digest16"]
    assert total_best == a["sum_best_pool"]


def test_fuzz_fixtures_on_device():
    fx = fuzz_fixtures()
    tas = []
    for f in fx:
        preset = M.PRESETS[f["seed"] % 6]
        s = f["seed"]
        tas.append(tracegen.synth_arrays(tracegen.SynthConfig.for_preset(
            preset, seed=s, num_layers=4 + s % 9, num_microbatches=1 + s % 4, transient_ratio=0.2 + (s % 5) * 0.2)))
    bp = api.plan_batch(tas, tracegen.C4_CANDIDATES)
    for t, (f, ta) in enumerate(zip(fx, tas)):
        s0, s1 = int(bp.batch.ev_off[t]), int(bp.batch.ev_off[t + 1])
        order = bp.order[s0:s1]
        order = order[ta.dyn[order] == 0]
        for c, p in enumerate(f["plans"]):
            assert ta.id[order].tolist() == p["ids"]
            assert bp.addr[c, s0:s1][order].tolist() == p["addrs"], (f["seed"], c)
            assert int(bp.stats[t * 4 + c, 9]) == p["pool_size"]
        tr = M.Trace.from_arrays(ta)
        plan, rmap = M.plan_trace(tr)
        assert [[list(k), e.t_lo, e.t_hi, [[iv.lo, iv.hi] for iv in e.space]] for k, e in rmap.entries.items()] == f["reuse"]
        for reuse in (True, False):
            rep, log = M.simulate(tr, plan.to_bundle(rmap), reuse=reuse)
            want = f[f"sim_reuse_{int(reuse)}"]
            assert rep.to_dict() == want["report"] and log_digest(log) == want["log_digest"]
        assert M.run_baseline(tr).to_dict() == f["baseline"]


@pytest.mark.slow
def test_app_b_c5_single_cta_layers(monkeypatch):
    """c5's one huge unit through the single-CTA layer kernel (the cooperative
    whole-GPU kernel k_layers_big switched off) gives the same plan file."""
    monkeypatch.setenv("STW_NO_BIG_COOP", "1")
    a = anchors()["c5_llama3_70b"]
    tr = M.Trace.from_arrays(tracegen.synth_arrays(tracegen.config("c5_llama3_70b")))
    plan, rmap = M.plan_trace(tr)
    assert hashlib.sha256(planio.dumps_plan(plan.to_bundle(rmap)).encode()).hexdigest()[:16] == a["write_plan_sha16"]


@pytest.mark.parametrize("name", ["c1_llama2_7b_1f1b", "c3_mixtral_moe", "c3b_mixtral_moe_rcp"])
def test_app_b_replay_general_warp(name, monkeypatch):
    """The general sequential replay warp (k_replay, forced) reproduces the
    reference's replay report, log digest and baseline report, like the
    register-resident warp the default path takes."""
    monkeypatch.setenv("STW_REPLAY_GENERAL", "1")
    a = anchors()[name]
    tr = M.Trace.from_arrays(tracegen.synth_arrays(tracegen.config(name)))
    plan, rmap = M.plan_trace(tr)
    rep, log = M.simulate(tr, plan.to_bundle(rmap))
    assert rep.to_dict() == a["sim"]
    assert log_digest(log) == a["sim_log_digest"]
    assert M.run_baseline(tr).to_dict() == a["baseline"]


@pytest.mark.parametrize("name", ["c3_mixtral_moe", "c3b_mixtral_moe_rcp"])
def test_app_b_simulate_full_chain(name, monkeypatch, capfd):
    """simulate takes the planned static allocations off the sequential chain
    when that is exact (replay_reg.cu: offchain_check); the full chain (forced)
    and the default give the reference's report and log digest."""
    a = anchors()[name]
    tr = M.Trace.from_arrays(tracegen.synth_arrays(tracegen.config(name)))
    plan, rmap = M.plan_trace(tr)
    bundle = plan.to_bundle(rmap)
    monkeypatch.setenv("STW_REPLAY_STATS", "1")
    rep, log = M.simulate(tr, bundle)
    assert "off-planned chain" in capfd.readouterr().err  # the default took the short chain here
    assert rep.to_dict() == a["sim"] and log_digest(log) == a["sim_log_digest"]
    monkeypatch.setenv("STW_REPLAY_FULL_CHAIN", "1")
    rep, log = M.simulate(tr, bundle)
    assert "full chain" in capfd.readouterr().err
    assert rep.to_dict() == a["sim"] and log_digest(log) == a["sim_log_digest"]


@pytest.mark.parametrize("chain", [True, False])
def test_app_b_c2_big_unit_resolve(chain, monkeypatch):
    """c2 is one unit too large for a warp's shared memory: the whole-GPU layer
    kernel resolves its gap classes by the parallel per-layer chain (default)
    or by the warp-serial resolve (STW_NO_CHAIN); both give the reference's plan."""
    if not chain:
        monkeypatch.setenv("STW_NO_CHAIN", "1")
    a = anchors()["c2_llama2_7b_vpp_rcp"]
    st = M.PlanStats()
    tr = M.Trace.from_arrays(tracegen.synth_arrays(tracegen.config("c2_llama2_7b_vpp_rcp")))
    plan, rmap = M.plan_trace(tr, stats=st)
    assert st.to_dict()["gap_insertions"] == a["stats"]["gap_insertions"]
    assert hashlib.sha256(planio.dumps_plan(plan.to_bundle(rmap)).encode()).hexdigest()[:16] == a["write_plan_sha16"]
