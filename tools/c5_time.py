"""Phase timings (STW_DEBUG_TIMING=2) of the c5 single-trace plan under the four candidates."""
import os
import sys
import time

sys.path.insert(0, "/root/repo")
from paper_2507_16274_b200 import api, tracegen  # noqa: E402

ta = tracegen.synth_arrays(tracegen.config("c5_llama3_70b"))
for it in range(3):
    if it == 2:
        os.environ["STW_DEBUG_TIMING"] = "2"
    t0 = time.perf_counter()
    bp = api.plan_batch([ta], tracegen.C4_CANDIDATES, select_best=True)
    print(f"plan c5 x4 candidates: {(time.perf_counter() - t0) * 1e3:.1f} ms", file=sys.stderr)
