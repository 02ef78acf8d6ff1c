"""Host-enqueue vs GPU-completion time per planner phase (STW_DEBUG_TIMING=2), device inputs."""
import ctypes as C
import os
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_2507_16274_b200 import _lib, api, tracegen  # noqa: E402
from paper_2507_16274_b200.batching import HostBatch  # noqa: E402

tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(4096)]
hb = HostBatch(tas)
db = hb.to_device("cuda")
L = _lib.load()
C4 = tracegen.C4_CANDIDATES
cb = api._cand_bits(C4)
T, N = hb.T, hb.N
o_rc = torch.empty(T * 4, dtype=torch.int32, device="cuda")
o_stats = torch.empty(T * 4 * _lib.NSTATS, dtype=torch.int64, device="cuda")
out = _lib.PlanOut(1, _lib.ptr(o_rc), None, _lib.ptr(o_stats), None, None, None, None, None, None, None, None, None,
                   None)
opts = _lib.PlanOpts(4, 1, _lib.ptr(cb), 512, C.c_void_p(torch.cuda.current_stream().cuda_stream))
st = db.struct()
err = _lib.errbuf()
for i in range(4):
    if i == 3:
        os.environ["STW_DEBUG_TIMING"] = "2"
    _lib.check(L.stw_plan_batch(C.byref(st), C.byref(opts), C.byref(out), err, 1024), err)
