"""Where one simulate / run_baseline call's time goes (kernels vs host), per config."""
import sys
import time

sys.path.insert(0, "/root/repo")
import paper_2507_16274_b200 as M  # noqa: E402
from paper_2507_16274_b200 import _lib, tracegen  # noqa: E402

for name in sys.argv[1:] or ["c3b_mixtral_moe_rcp"]:
    tr = M.Trace.from_arrays(tracegen.synth_arrays(tracegen.config(name)))
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
        print(f"{name} {what}: wall {wall:.2f} ms, kernels {tot:.2f} ms ({sum(v[0] for v in prof.values())} launches):",
              ", ".join(f"{k} {v[1]:.2f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]))
