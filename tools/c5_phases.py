"""Phase timing (STW_DEBUG_TIMING=2) and per-kernel times of one c5 planner call."""
import os
import sys

sys.path.insert(0, "/root/repo")
from paper_2507_16274_b200 import _lib, api, tracegen  # noqa: E402

ta = tracegen.synth_arrays(tracegen.config(sys.argv[1] if len(sys.argv) > 1 else "c5_llama3_70b"))
api.plan_batch([ta], ((True, True),), detail=False)
os.environ["STW_DEBUG_TIMING"] = "2"
_lib.profile(True)
api.plan_batch([ta], ((True, True),), detail=False)
_lib.profile(False)
for k, (c, ms) in sorted(_lib.profile_collect().items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {k:24s} x{c:4d} {ms:9.3f} ms")
