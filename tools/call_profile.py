"""Where one planner call's time goes: per-kernel device time (libstw's
event profiler) vs the call's wall time, for a c4 batch of T traces (device-
resident inputs and outputs, as in bench.py).  python tools/call_profile.py T"""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_16274_b200 import _lib, api  # noqa: E402
from paper_2507_16274_b200.batching import HostBatch  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dev = torch.device("cuda", 0)
hb = HostBatch(bench.make_traces(range(T)), pinned=True)
db = hb.to_device(dev)
Cn = 4
L = _lib.load()
cb = api._cand_bits(bench.CANDS)
s = torch.cuda.current_stream(dev)
o = {k: torch.empty(n, dtype=dt, device=dev) for k, n, dt in (
    ("rc", T * Cn, torch.int32), ("err", 2 * T * Cn, torch.int64), ("stats", T * Cn * _lib.NSTATS, torch.int64),
    ("best", T, torch.int32), ("bpool", T, torch.int64), ("abest", hb.N, torch.int64))}
addr = torch.empty((Cn, hb.N), dtype=torch.int64, device=dev)
out = _lib.PlanOut(1, _lib.ptr(o["rc"]), _lib.ptr(o["err"]), _lib.ptr(o["stats"]), _lib.ptr(addr), None, None, None,
                   None, None, None, _lib.ptr(o["best"]), _lib.ptr(o["abest"]), _lib.ptr(o["bpool"]))
opts = _lib.PlanOpts(Cn, 1, _lib.ptr(cb), 512, C.c_void_p(s.cuda_stream))
b = db.struct()
err = _lib.errbuf()


def call():
    _lib.check(L.stw_plan_batch(C.byref(b), C.byref(opts), C.byref(out), err, 1024), err)


for _ in range(5):
    call()
torch.cuda.synchronize()
K = 20
t0 = time.perf_counter()
for _ in range(K):
    call()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K * 1e3
_lib.profile_collect(reset=True)
_lib.profile(True)
for _ in range(K):
    call()
torch.cuda.synchronize()
_lib.profile(False)
prof = _lib.profile_collect(reset=True)
tot = sum(v[1] for v in prof.values()) / K
print(f"T={T}: wall {wall:.3f} ms/call; kernel time (sum of launches, event-timed) {tot:.3f} ms; "
      f"launches/call {sum(v[0] for v in prof.values()) / K:.0f}")
for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {k:34s} {c / K:5.1f}/call {ms / K * 1e3:9.1f} us/call")
