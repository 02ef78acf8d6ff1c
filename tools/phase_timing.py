"""Host enqueue vs GPU completion per planner phase for the c4 batch (developer aid):
STW_DEBUG_TIMING=2 on the last of a few warm calls. python tools/phase_timing.py"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2507_16274_b200 import api, tracegen  # noqa: E402
from paper_2507_16274_b200.batching import HostBatch  # noqa: E402

tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(4096)]
hb = HostBatch(tas, pinned=True)

for _ in range(3):
    api.plan_batch(hb, tracegen.C4_CANDIDATES, select_best=True, detail=False)
torch.cuda.synchronize()
os.environ["STW_DEBUG_TIMING"] = "2"
api.plan_batch(hb, tracegen.C4_CANDIDATES, select_best=True, detail=False)
torch.cuda.synchronize()
