import os
import sys

sys.path.insert(0, "/root/repo")
os.environ["STW_DEBUG_DUMP"] = "1"
from paper_2507_16274_b200 import api, tracegen  # noqa: E402

sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/tools")
from test_gpu_plan import fuzz_cfg  # noqa: E402

ta = tracegen.synth_arrays(fuzz_cfg(0))
bp = api.plan_batch([ta], ((True, False),))
print(bp.addr[0] >> 20)
