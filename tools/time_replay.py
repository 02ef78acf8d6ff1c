"""simulate / run_baseline per config on the device (best of 3) beside the C
port of the reference (1 host thread), plus bit-exactness of the reports."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2507_16274_b200 as M  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2507_16274_b200 import tracegen  # noqa: E402


def best(fn, k=3):
    t, r = 1e9, None
    for _ in range(k):
        t0 = time.perf_counter()
        r = fn()
        t = min(t, time.perf_counter() - t0)
    return t * 1e3, r


names = [a for a in sys.argv[1:] if not a.startswith("-")] or ["c1_llama2_7b_1f1b", "c2_llama2_7b_vpp_rcp", "c3_mixtral_moe", "c3b_mixtral_moe_rcp",
                         "c5_llama3_70b"]
for name in names:
    ta = tracegen.synth_arrays(tracegen.config(name))
    tr = M.Trace.from_arrays(ta)
    plan, rmap = M.plan_trace(tr)
    bundle = plan.to_bundle(rmap)
    c = plan.columns()
    keys, kidx = ta.dynamic_keys()
    off, lo, hi = O.reuse(c.addr, c.size, c.t_s, c.t_e, [rmap.entries[k].t_lo for k in keys],
                          [rmap.entries[k].t_hi for k in keys])
    ts, (rep, _) = best(lambda: M.simulate(tr, bundle))
    tb, base = best(lambda: M.run_baseline(tr))
    key = np.where(kidx >= 0, kidx, -1).astype(np.int32)
    cs, orep = best(lambda: O.simulate(ta, key, plan.pool_size, 512, c.id, c.addr, c.size, c.t_s, c.t_e, off, lo, hi,
                                       True), 1)
    cb, obase = best(lambda: O.baseline(ta), 1)
    ok = orep.report == rep.to_dict() and obase.report == base.to_dict()
    print(f"{name:22s} simulate {ts:8.2f} ms (cpu {cs:8.2f})  baseline {tb:8.2f} ms (cpu {cb:8.2f})  exact={ok}")

if "--prof" in sys.argv or True:
    from paper_2507_16274_b200 import _lib

    for name in names[:1] + (["c2_llama2_7b_vpp_rcp"] if "c2_llama2_7b_vpp_rcp" in names else []):
        ta = tracegen.synth_arrays(tracegen.config(name))
        tr = M.Trace.from_arrays(ta)
        plan, rmap = M.plan_trace(tr)
        bundle = plan.to_bundle(rmap)
        for what, fn in (("simulate", lambda: M.simulate(tr, bundle)), ("baseline", lambda: M.run_baseline(tr))):
            fn()
            _lib.profile_collect(reset=True)
            _lib.profile(True)
            t0 = time.perf_counter()
            fn()
            wall = (time.perf_counter() - t0) * 1e3
            _lib.profile(False)
            prof = _lib.profile_collect(reset=True)
            tot = sum(v[1] for v in prof.values())
            print(f"{name} {what}: wall {wall:.2f} ms, kernels {tot:.2f} ms:",
                  ", ".join(f"{k} {v[1]:.2f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:6]))
