"""One c5 planner call (4 candidates) for ncu captures."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2507_16274_b200 import api, tracegen  # noqa: E402
ta = tracegen.synth_arrays(tracegen.config("c5_llama3_70b"))
api.plan_batch([ta], tracegen.C4_CANDIDATES, select_best=True)
