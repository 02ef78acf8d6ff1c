"""Drive libstw_alloc as torch's CUDA allocator: replay a small MoE trace's
requests as real tensors and check every static tensor lands at its planned
offset inside the reserved pool."""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_16274_b200 as M  # noqa: E402
from paper_2507_16274_b200 import tracegen  # noqa: E402
from paper_2507_16274_b200.runtime import PlanAllocator  # noqa: E402

ta = tracegen.synth_arrays(tracegen.SynthConfig.for_preset("moe_recompute", seed=1, num_layers=4, num_microbatches=2))
tr = M.Trace.from_arrays(ta)
plan, rmap = M.plan_trace(tr)  # planning runs on the device via libstw
bundle = plan.to_bundle(rmap)
rt = PlanAllocator(bundle, tr)
PlanAllocator.install()
n = len(ta)
t = np.concatenate([ta.t_s, ta.t_e])
is_alloc = np.concatenate([np.ones(n, np.int64), np.zeros(n, np.int64)])
ids = np.concatenate([ta.id, ta.id])
names, kidx = ta.dynamic_keys()
live = {}
planned = {int(i): int(a) for i, a in zip(bundle._cols.id, bundle._cols.addr)}
checked = 0
for o in np.lexsort((ids, is_alloc, t)).tolist():
    e = o % n
    if is_alloc[o]:
        if ta.dyn[e]:
            rt.set_layer(names[kidx[e]], True)
        else:
            rt.set_layer(None, False)
            rt.set_phase(int(ta.ps[e]))
        x = torch.empty(int(ta.size[e]), dtype=torch.uint8, device="cuda")
        x.fill_(e % 251)
        live[e] = x
        v, route = PlanAllocator.vaddr(x.data_ptr())
        if route == "planned":
            assert v == planned[int(ta.id[e])], (e, v)
            checked += 1
        del x  # the trace's free must release the last tensor too
    else:
        del live[e]
torch.cuda.synchronize()
rep = PlanAllocator.report()
print(f"torch pluggable allocator ok: {checked} planned tensors at their offsets, frag {rep.fragmentation:.4f}")
