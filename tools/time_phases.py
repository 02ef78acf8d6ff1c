import os, sys, time
sys.path.insert(0, "/root/repo")
from paper_2507_16274_b200 import api, tracegen
from paper_2507_16274_b200.batching import HostBatch
tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(4096)]
hb = HostBatch(tas)
C4 = tracegen.C4_CANDIDATES
for i in range(3):
    api.plan_batch(hb, C4, select_best=True, detail=False)
os.environ["STW_DEBUG_TIMING"] = "1"
t = time.perf_counter(); api.plan_batch(hb, C4, select_best=True, detail=False); print("total", time.perf_counter() - t)
