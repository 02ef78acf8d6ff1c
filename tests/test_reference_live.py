"""Live cross-checks against the reference package (build container only;
skipped where /root/reference is absent, e.g. on the GPU box)."""

import random

import numpy as np
import pytest

from conftest import ref
from paper_2507_16274_b200 import soa, tracegen
from oracle import oracle as O


def test_tracegen_reproduces_reference_synth():
    R = ref()
    rng = random.Random(11)
    for i in range(40):
        preset = tracegen.PRESETS[i % 6]
        kw = dict(num_layers=rng.randint(2, 10), num_microbatches=rng.randint(1, 5),
                  transient_ratio=rng.choice([0.0, 0.3, 1.0, 2.5]), seed=rng.randint(0, 10**6))
        if "vpp" in preset:
            kw["num_chunks"] = rng.randint(2, min(3, kw["num_layers"]))
        rt = R.synth_trace(R.SynthConfig.for_preset(preset, **kw))
        mine = tracegen.synth_arrays(tracegen.SynthConfig.for_preset(preset, **kw))
        other = soa.from_trace(rt)
        for f in ("id", "size", "t_s", "t_e", "ps", "pe", "dyn", "ls", "le", "phase_start", "phase_end"):
            assert np.array_equal(getattr(mine, f), getattr(other, f)), (preset, f)
        assert mine.layer_names == other.layer_names


def test_oracle_matches_reference_random_traces():
    R = ref()
    from memplan.planner import PlanStats

    rng = random.Random(5)
    for i in range(30):
        preset = tracegen.PRESETS[i % 6]
        cfg = R.SynthConfig.for_preset(preset, seed=rng.randint(0, 10**6), num_layers=rng.randint(3, 9),
                                       num_microbatches=rng.randint(1, 4), transient_ratio=rng.random() * 2)
        rt = R.synth_trace(cfg)
        ta = soa.from_trace(rt)
        for f, g in tracegen.C4_CANDIDATES:
            st = PlanStats()
            rp = R.synthesize_static_plan(rt, fusion=f, gap_insert=g, stats=st)
            op = O.plan(ta, f, g)
            assert {d.id: d.addr for d in rp.decisions} == {int(ta.id[k]): int(op.addr[k]) for k in np.nonzero(ta.dyn == 0)[0]}
            assert st.accepted_fusions == op.accepted


def test_oracle_validate_matches_reference_on_invalid_plans():
    R = ref()
    from memplan.model import AllocationDecision, MemoryRequestEvent, PhaseId
    from memplan.planner import StaticPlan

    rng = random.Random(3)
    F, B = PhaseId.parse("F:0"), PhaseId.parse("B:0")
    for _ in range(200):
        evs = []
        for i in range(rng.randint(1, 25)):
            s = rng.randint(0, 20)
            evs.append(MemoryRequestEvent(i * 3 + 1, 512 * rng.randint(1, 8), s, s + rng.randint(1, 10), F, B))
        decs = tuple(AllocationDecision(e, 512 * rng.randint(0, 20)) for e in evs)
        want = [(a.id, b.id) for a, b in R.validate_plan(StaticPlan(1 << 30, 512, decs, (), 0))]
        n, pairs = O.validate([d.id for d in decs], [d.addr for d in decs], [d.size for d in decs],
                              [d.t_s for d in decs], [d.t_e for d in decs])
        assert want == [(decs[a].id, decs[b].id) for a, b in pairs]
