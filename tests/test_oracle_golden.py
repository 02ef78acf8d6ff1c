"""Pin the C oracle (and the trace generator) to the reference's own outputs.

Fixtures in tests/golden/ were produced by running the REFERENCE package
(make_golden.py); these tests need no reference and no GPU."""

import numpy as np
import pytest

from paper_2507_16274_b200 import tracegen
from oracle import oracle as O

from _util import (anchors, fuzz_fixtures, log_digest, oracle_log_dicts, plan_sha16, reuse_windows, static_order,
                   trace_digest)

STATS = {"events": "num_events", "persistent": "num_persistent", "phase_groups": "num_groups",
         "local_plans": "num_plans", "residual_events": "num_residuals", "fusion_attempts": "fusion_attempts",
         "fusion_accepted": "fusion_accepted", "gap_insertions": "gap_insertions", "layers": "num_layers",
         "pool_size": "pool_size", "static_peak": "static_peak"}


def fuzz_cfg(seed):
    preset = tracegen.PRESETS[seed % 6]
    return tracegen.SynthConfig.for_preset(preset, seed=seed, num_layers=4 + seed % 9,
                                          num_microbatches=1 + seed % 4, transient_ratio=0.2 + (seed % 5) * 0.2)


def full_check(ta, fx_plan=None, anchor=None):
    """Plan + reuse + replay + baseline through the oracle; compare to a fixture or anchor."""
    r = O.plan(ta, True, True)
    assert r.rc == 0, r.err
    order = static_order(ta)
    keys, t_lo, t_hi = reuse_windows(ta)
    off, lo, hi = O.reuse(r.addr[order], ta.size[order], ta.t_s[order], ta.t_e[order], t_lo, t_hi)
    spaces = [list(zip(lo[off[k]:off[k + 1]].tolist(), hi[off[k]:off[k + 1]].tolist())) for k in range(len(keys))]
    names, kidx = ta.dynamic_keys()
    key = np.where(kidx >= 0, kidx, -1).astype(np.int32)
    sims = {}
    for reuse in (True, False):
        s = O.simulate(ta, key, r.stats["pool_size"], 512, ta.id[order], r.addr[order], ta.size[order],
                       ta.t_s[order], ta.t_e[order], off, lo, hi, reuse)
        assert s.rc == 0, s.err
        sims[reuse] = s
    b = O.baseline(ta)
    sha = plan_sha16(r.stats["pool_size"], 512, ta.id[order], r.addr[order], ta.size[order], ta.t_s[order],
                     ta.t_e[order], list(zip(keys, spaces)))
    return r, keys, spaces, sims, b, sha


def test_fuzz_fixtures_plan_all_candidates():
    for fx in fuzz_fixtures():
        ta = tracegen.synth_arrays(fuzz_cfg(fx["seed"]))
        assert trace_digest(ta) == fx["trace_digest"]
        order = static_order(ta)
        for p in fx["plans"]:
            r = O.plan(ta, p["fusion"], p["gap_insert"])
            assert r.rc == 0
            assert ta.id[order].tolist() == p["ids"]
            assert r.addr[order].tolist() == p["addrs"]
            assert r.stats["pool_size"] == p["pool_size"]
            assert r.stats["persistent_size"] == p["persistent_size"]
            for k, v in p["stats"].items():
                if k in STATS:
                    assert r.stats[STATS[k]] == v, (fx["seed"], k)
            assert [list(x) for x in r.accepted] == p["accepted_fusions"]
            assert [[int(b), int(s)] for b, s in zip(r.layer_base, r.layer_size)] == p["layer_table"]


def test_fuzz_fixtures_reuse_replay_baseline():
    for fx in fuzz_fixtures():
        ta = tracegen.synth_arrays(fuzz_cfg(fx["seed"]))
        r, keys, spaces, sims, b, _ = full_check(ta)
        assert [[list(k), [list(iv) for iv in sp]] for k, sp in zip(keys, spaces)] == \
            [[k, ivs] for k, _, _, ivs in fx["reuse"]]
        for reuse in (True, False):
            want = fx[f"sim_reuse_{int(reuse)}"]
            got = sims[reuse]
            assert got.report == want["report"], (fx["seed"], reuse)
            assert log_digest(oracle_log_dicts(got.log, ta)) == want["log_digest"]
        assert b.report == fx["baseline"]
        assert O.peak_live(ta.size, ta.t_s, ta.t_e) == fx["clique_lower_bound"]


@pytest.mark.parametrize("name", ["c1_llama2_7b_1f1b", "c3_mixtral_moe", "c3b_mixtral_moe_rcp", "c2_llama2_7b_vpp_rcp"])
def test_app_b_anchors(name):
    a = anchors()[name]
    ta = tracegen.synth_arrays(tracegen.config(name))
    assert trace_digest(ta) == a["trace_digest"]
    assert (len(ta), ta.horizon, ta.n_sched) == (a["events"], a["horizon"], a["phases"])
    r, keys, spaces, sims, b, sha = full_check(ta)
    assert r.stats["pool_size"] == a["pool_size"] and r.stats["static_peak"] == a["static_peak"]
    for k, v in a["stats"].items():
        if k in STATS:
            assert r.stats[STATS[k]] == v, k
    assert sha == a["write_plan_sha16"]
    assert sims[True].report == a["sim"]
    assert log_digest(oracle_log_dicts(sims[True].log, ta)) == a["sim_log_digest"]
    assert b.report == a["baseline"]
    assert O.peak_live(ta.size, ta.t_s, ta.t_e) == a["clique_lower_bound"]


@pytest.mark.slow
def test_app_b_c5_anchor():
    test_app_b_anchors("c5_llama3_70b")


def test_c4_digest_sample_lines():
    """The first c4 lines of the digest recipe from the oracle."""
    import hashlib

    a = anchors()["c4"]
    for line in a["lines_sha_first8"]:
        seed = int(line.split("|")[0])
        ta = tracegen.synth_arrays(tracegen.c4_config(seed))
        order = static_order(ta)
        parts, pools = [], []
        for f, g in tracegen.C4_CANDIDATES:
            r = O.plan(ta, f, g)
            h8 = hashlib.sha256(",".join(f"{i}:{x}" for i, x in zip(ta.id[order].tolist(),
                                                                  r.addr[order].tolist())).encode()).hexdigest()[:8]
            parts.append(f"{r.stats['pool_size']}:{h8}")
            pools.append(r.stats["pool_size"])
        best = min(range(4), key=lambda c: (pools[c], c))
        assert f"{seed}|{len(order)}|{best}|" + "|".join(parts) == line
