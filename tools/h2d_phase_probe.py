import torch, time, sys, os
sys.path.insert(0, "/root/repo")
x = torch.empty(46_500_000, dtype=torch.uint8).pin_memory(); y = torch.empty_like(x, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): y.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/10
print(f"H2D 46.5 MB: {ms:.3f} ms = {46.5/ms:.1f} GB/s")
z = torch.empty(13_200_000, dtype=torch.uint8).pin_memory(); w = torch.empty_like(z, device="cuda")
e0.record()
for _ in range(10): z.copy_(w, non_blocking=True)
e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/10
print(f"D2H 13.2 MB: {ms:.3f} ms = {13.2/ms:.1f} GB/s")
import bench
from paper_2507_16274_b200 import api
from paper_2507_16274_b200.batching import HostBatch
hb = HostBatch(bench.make_traces(range(4096)), pinned=True)
api.plan_batch(hb, bench.CANDS, select_best=True, detail=False)
os.environ["STW_DEBUG_TIMING"] = "2"
api.plan_batch(hb, bench.CANDS, select_best=True, detail=False)
