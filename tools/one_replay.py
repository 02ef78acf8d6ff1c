"""One replay call for ncu: python tools/one_replay.py <config> simulate|baseline"""
import sys

sys.path.insert(0, ".")
import paper_2507_16274_b200 as M  # noqa: E402
from paper_2507_16274_b200 import tracegen  # noqa: E402

name, what = sys.argv[1], sys.argv[2]
tr = M.Trace.from_arrays(tracegen.synth_arrays(tracegen.config(name)))
if what == "baseline":
    M.run_baseline(tr)
else:
    plan, rmap = M.plan_trace(tr)
    M.simulate(tr, plan.to_bundle(rmap))
