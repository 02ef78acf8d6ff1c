"""c5 through the package API (synthesize_static_plan), with the library's phase
timing on the last call: where the end-to-end time beyond the kernels goes."""
import os
import sys
import time

sys.path.insert(0, "/root/repo")
import paper_2507_16274_b200 as M  # noqa: E402
from paper_2507_16274_b200 import tracegen  # noqa: E402

tr = M.Trace.from_arrays(tracegen.synth_arrays(tracegen.config("c5_llama3_70b")))
for it in range(3):
    if it == 2:
        os.environ["STW_DEBUG_TIMING"] = "2"
    t0 = time.perf_counter()
    plan = M.synthesize_static_plan(tr)
    t1 = time.perf_counter()
    c = plan.columns()
    t2 = time.perf_counter()
    print(f"synthesize_static_plan {1e3 * (t1 - t0):.1f} ms, columns {1e3 * (t2 - t1):.1f} ms", file=sys.stderr)
