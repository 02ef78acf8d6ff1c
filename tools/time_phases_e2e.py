"""Planner phase timings (STW_DEBUG_TIMING=2) inside the pipelined host-batch
call (stw_plan_batches), next to the device-input call: where the e2e gap goes."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_16274_b200 import _lib, api, tracegen  # noqa: E402
from paper_2507_16274_b200.batching import HostBatch  # noqa: E402

tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(4096)]
hb = HostBatch(tas, pinned=True)
T, N = hb.T, hb.N
L = _lib.load()
C4 = tracegen.C4_CANDIDATES
cb = api._cand_bits(C4)
pin = lambda n, dt: torch.empty(n, dtype=dt).pin_memory().numpy()  # noqa: E731
h_rc, h_err, h_stats = pin(T * 4, torch.int32), pin(2 * T * 4, torch.int64), pin(T * 4 * _lib.NSTATS, torch.int64)
h_best, h_abest, h_bpool = pin(T, torch.int32), pin(N, torch.int64), pin(T, torch.int64)
out = _lib.PlanOut(0, _lib.ptr(h_rc), _lib.ptr(h_err), _lib.ptr(h_stats), None, None, None, None, None, None, None,
                   _lib.ptr(h_best), _lib.ptr(h_abest), _lib.ptr(h_bpool))
stream = torch.cuda.current_stream()
opts = _lib.PlanOpts(4, 1, _lib.ptr(cb), 512, C.c_void_p(stream.cuda_stream))
st = hb.struct()
err = _lib.errbuf()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
bs = (_lib.Batch * k)(*([st] * k))
os_ = (_lib.PlanOut * k)(*([out] * k))
serial = len(sys.argv) > 2 and sys.argv[2] == "serial"
for it in range(3):
    if it == 2:
        os.environ["STW_DEBUG_TIMING"] = "2"
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if serial:
        for _ in range(k):
            _lib.check(L.stw_plan_batch(C.byref(st), C.byref(opts), C.byref(out), err, 1024), err)
    else:
        _lib.check(L.stw_plan_batches(k, bs, C.byref(opts), os_, err, 1024), err)
    torch.cuda.synchronize()
    print(f"{'serial' if serial else 'plan_batches'} k={k}: {(time.perf_counter() - t0) * 1e3 / k:.3f} ms/batch",
          file=sys.stderr)
