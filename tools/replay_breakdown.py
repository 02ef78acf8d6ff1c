"""Wall time of one replay API call vs its kernels (developer aid).
python tools/replay_breakdown.py <config> simulate|baseline [reps]
Under ncu (--nvtx --nvtx-include timed/) the last call's launches are selected."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2507_16274_b200 as M  # noqa: E402
from paper_2507_16274_b200 import tracegen  # noqa: E402

name, what = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
tr = M.Trace.from_arrays(tracegen.synth_arrays(tracegen.config(name)))
if what == "baseline":
    fn = lambda: M.run_baseline(tr)  # noqa: E731
else:
    plan, rmap = M.plan_trace(tr)
    bundle = plan.to_bundle(rmap)
    fn = lambda: M.simulate(tr, bundle)  # noqa: E731
fn()
best = float("inf")
for _ in range(reps):
    t0 = time.perf_counter()
    fn()
    best = min(best, time.perf_counter() - t0)
torch.cuda.nvtx.range_push("timed")
fn()
torch.cuda.nvtx.range_pop()
print(f"{name} {what}: best wall {best * 1e3:.3f} ms")
