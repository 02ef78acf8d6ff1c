"""Generate the parity fixtures from the REFERENCE implementation (run in the
build container, where /root/reference exists; the outputs are committed so the
GPU box -- which has no reference -- can pin against them).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes:
  anchors.json     App. B anchors per pinned config + the c4 digest
  fuzz.json.gz     reference outputs for 48 small fuzz traces (test_acceptance.py:28-36
                   generator): plan addresses per candidate, PlanStats, accepted
                   fusions, reuse map, simulate report + log digest, baseline report
"""

from __future__ import annotations

import gzip
import hashlib
import json
import multiprocessing as mp
import os
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

import memplan as R  # noqa: E402
from memplan.planner import PlanStats  # noqa: E402

MIB = 1 << 20
L2 = tuple(n * MIB for n in (32, 96, 86, 172))
MX = tuple(n * MIB for n in (32, 48, 112))
L3 = tuple(n * MIB for n in (16, 20, 56, 112))
MOE = dict(num_layers=32, num_microbatches=64, transient_ratio=1.0, size_palette=MX, distinct_sizes=3,
           persistent_bytes=16384 * MIB, moe_size_range=(4 * MIB, 56 * MIB))
CFGS = {
    "c1_llama2_7b_1f1b": ("dense", dict(num_layers=16, num_microbatches=96, transient_ratio=2.0, size_palette=L2,
                                        distinct_sizes=4, persistent_bytes=8192 * MIB)),
    "c2_llama2_7b_vpp_rcp": ("dense_vpp_recompute", dict(num_layers=32, num_chunks=2, num_microbatches=448,
                                                         transient_ratio=2.0, size_palette=L2, distinct_sizes=4,
                                                         persistent_bytes=16384 * MIB)),
    "c3_mixtral_moe": ("moe", dict(MOE)),
    "c3b_mixtral_moe_rcp": ("moe_recompute", dict(MOE)),
    "c5_llama3_70b": ("dense_vpp_recompute", dict(num_layers=80, num_chunks=4, num_microbatches=1024,
                                                  transient_ratio=4.5, size_palette=L3, distinct_sizes=4,
                                                  persistent_bytes=20480 * MIB)),
}
C4 = ("dense", "dense_recompute", "dense_vpp", "dense_vpp_recompute")
CANDS = ((True, True), (True, False), (False, True), (False, False))


def sha(data: bytes) -> str:
    return hashlib.sha256(data).hexdigest()


def trace_digest(tr) -> str:
    h = hashlib.sha256()
    for e in tr.events:
        h.update(f"{e.id},{e.size},{e.t_s},{e.t_e},{e.p_s.tag()},{e.p_e.tag()},{int(e.dynamic)},{e.l_s},{e.l_e};".encode())
    for s in tr.phase_schedule:
        h.update(f"{s.phase.tag()},{s.start},{s.end};".encode())
    for s in tr.layer_schedule:
        h.update(f"{s.name},{s.start},{s.end};".encode())
    return h.hexdigest()[:16]


def log_digest(log) -> str:
    return sha("\n".join(json.dumps(r, sort_keys=True, separators=(",", ":")) for r in log).encode())[:16]


def anchor(name):
    preset, kw = CFGS[name]
    tr = R.synth_trace(R.SynthConfig.for_preset(preset, seed=0, **kw))
    st = PlanStats()
    plan, rmap = R.plan_trace(tr, stats=st)
    bundle = plan.to_bundle(rmap)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "plan.json")
        R.write_plan(bundle, p)
        plan_sha = sha(open(p, "rb").read())[:16]
    rep, log = R.simulate(tr, bundle)
    base = R.run_baseline(tr)
    return name, {
        "trace_digest": trace_digest(tr), "events": len(tr.events), "horizon": tr.horizon,
        "phases": len(tr.phase_schedule), "pool_size": plan.pool_size, "static_peak": st.static_peak,
        "stats": st.to_dict() | {"plan_seconds": None}, "accepted_fusions": st.accepted_fusions,
        "clique_lower_bound": R.clique_lower_bound(tr),
        "reuse_keys": len(rmap.entries), "reuse_intervals": sum(len(e.space) for e in rmap.entries.values()),
        "write_plan_sha16": plan_sha, "sim": rep.to_dict(), "sim_log_digest": log_digest(log),
        "baseline": base.to_dict(),
    }


def c4_line(seed: int) -> str:
    cfg = R.SynthConfig.for_preset(C4[seed % 4], seed=seed, num_layers=4 + seed % 29,
                                   num_microbatches=1 + seed % 8, transient_ratio=0.2 + (seed % 5) * 0.2)
    tr = R.synth_trace(cfg)
    parts = []
    pools = []
    for f, g in CANDS:
        p = R.synthesize_static_plan(tr, fusion=f, gap_insert=g)
        h8 = sha(",".join(f"{d.id}:{d.addr}" for d in p.decisions).encode())[:8]
        parts.append(f"{p.pool_size}:{h8}")
        pools.append(p.pool_size)
    best = min(range(4), key=lambda c: (pools[c], c))
    n = len(tr.static_events())
    return f"{seed}|{n}|{best}|" + "|".join(parts) + "\n"


def fuzz_case(seed: int):
    preset = R.PRESETS[seed % 6]
    cfg = R.SynthConfig.for_preset(preset, seed=seed, num_layers=4 + seed % 9, num_microbatches=1 + seed % 4,
                                   transient_ratio=0.2 + (seed % 5) * 0.2)
    tr = R.synth_trace(cfg)
    out = {"seed": seed, "preset": preset, "trace_digest": trace_digest(tr), "plans": []}
    for f, g in CANDS:
        st = PlanStats()
        p = R.synthesize_static_plan(tr, fusion=f, gap_insert=g, stats=st)
        out["plans"].append({
            "fusion": f, "gap_insert": g, "pool_size": p.pool_size, "persistent_size": p.persistent_size,
            "ids": [d.id for d in p.decisions], "addrs": [d.addr for d in p.decisions],
            "layer_table": [[b, l.size] for b, l in p.layer_table],
            "stats": st.to_dict() | {"plan_seconds": None}, "accepted_fusions": st.accepted_fusions,
        })
    plan, rmap = R.plan_trace(tr)
    out["reuse"] = [[list(k), e.t_lo, e.t_hi, [[iv.lo, iv.hi] for iv in e.space]]
                    for k, e in sorted(rmap.entries.items())]
    bundle = plan.to_bundle(rmap)
    for reuse in (True, False):
        rep, log = R.simulate(tr, bundle, reuse=reuse)
        out[f"sim_reuse_{int(reuse)}"] = {"report": rep.to_dict(), "log_digest": log_digest(log), "log_len": len(log)}
    out["baseline"] = R.run_baseline(tr).to_dict()
    out["clique_lower_bound"] = R.clique_lower_bound(tr)
    return out


def main():
    with mp.Pool(os.cpu_count()) as pool:
        fuzz = pool.map(fuzz_case, range(48))
        with gzip.open(os.path.join(HERE, "fuzz.json.gz"), "wt") as fh:
            json.dump(fuzz, fh)
        print("fuzz done", flush=True)
        anchors = dict(pool.map(anchor, list(CFGS)))
        lines = pool.map(c4_line, range(4096), chunksize=16)
    h = hashlib.sha256("".join(lines).encode()).hexdigest()[:16]
    total_best = sum(int(ln.split("|")[3 + int(ln.split("|")[2])].split(":")[0]) for ln in lines)
    anchors["c4"] = {"digest16": h, "sum_best_pool": total_best,
                     "static_events": sum(int(ln.split("|")[1]) for ln in lines),
                     "lines_sha_first8": [ln.strip() for ln in lines[:8]]}
    with open(os.path.join(HERE, "anchors.json"), "w") as fh:
        json.dump(anchors, fh, indent=1, sort_keys=True)
    print(json.dumps({k: (v.get("pool_size"), v.get("write_plan_sha16"), v.get("digest16")) for k, v in anchors.items()}))


if __name__ == "__main__":
    main()
