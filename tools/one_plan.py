"""One batched c4 planner call (for ncu captures)."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2507_16274_b200 import api, tracegen
from paper_2507_16274_b200.batching import HostBatch

tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(4096)]
hb = HostBatch(tas)
for _ in range(2):
    bp = api.plan_batch(hb, tracegen.C4_CANDIDATES, select_best=True, detail=False)
print("rc max", bp.rc.max())
