"""A small workload touching every libstw kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): K2 radix sort and the look-back scan over
many tiles, the batched planner (all candidates), K7, K8, K9/K10 replays, K1
the sub-operation kernels, the general replay warp, and
c2 (the cooperative huge-unit layer kernel, the exact validator). Each result is checked against the oracle, so a
race that changes a result fails here too.
    compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_16274_b200 as M  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2507_16274_b200 import api, planner, tracegen  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
n = 1 << 20  # ~270 onesweep tiles, ~256 scan tiles
keys = torch.randint(0, 1 << 40, (n,), dtype=torch.int64, device=dev, generator=g)
vals = torch.arange(n, dtype=torch.int32, device=dev)
ref = torch.sort(keys, stable=True)
api.radix_sort_pairs(keys, vals, 0, 40)
assert torch.equal(keys, ref.values) and torch.equal(vals.long(), ref.indices), "radix sort"
tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(48)]
bp = api.plan_batch(tas, tracegen.C4_CANDIDATES, select_best=True)
for t in range(0, 48, 7):
    s0, s1 = int(bp.batch.ev_off[t]), int(bp.batch.ev_off[t + 1])
    for c, (f, gi) in enumerate(tracegen.C4_CANDIDATES):
        r = O.plan(tas[t], f, gi)
        st = tas[t].dyn == 0
        assert np.array_equal(bp.addr[c, s0:s1][st], r.addr[st]), ("plan", t, c)
for name in ("c1_llama2_7b_1f1b", "c3_mixtral_moe"):
    ta = tracegen.synth_arrays(tracegen.config(name))
    tr = M.Trace.from_arrays(ta)
    plan, rmap = M.plan_trace(tr)
    rep, _ = M.simulate(tr, plan.to_bundle(rmap))
    base = M.run_baseline(tr)
    assert base.to_dict() == O.baseline(ta).report, name
    assert M.validate_plan(plan) == [] and M.peak_live_bytes(ta) == O.peak_live(ta.size, ta.t_s, ta.t_e)
# the general replay warp (forced), and c2: one unit too large for a warp's
# shared memory -> the cooperative whole-GPU layer kernel, and > 65 K
# rectangles -> the exact tiled validator with long-span live lists
import os  # noqa: E402

os.environ["STW_REPLAY_GENERAL"] = "1"
ta = tracegen.synth_arrays(tracegen.config("c1_llama2_7b_1f1b"))
assert M.run_baseline(M.Trace.from_arrays(ta)).to_dict() == O.baseline(ta).report, "general replay"
del os.environ["STW_REPLAY_GENERAL"]
ta = tracegen.synth_arrays(tracegen.config("c2_llama2_7b_vpp_rcp"))
r = O.plan(ta, True, True)
bp2 = api.plan_batch([ta], ((True, True),))
st = ta.dyn == 0
assert np.array_equal(bp2.addr[0][st], r.addr[st]), "c2 plan"
ev = [M.MemoryRequestEvent(i, (1 + i % 5) * 512, i, i + 3 + i % 4, M.PhaseId.parse("F:0"), M.PhaseId.parse("B:0"))
      for i in range(300)]
groups = planner.group_by_phase(ev)
plans = planner.pack_groups(groups)
items = [planner._Item(512, e.t_s, e.t_e, e.id, e) for e in ev]
assert len(planner.build_layers_for_size(items)) >= 1
# the concurrent paths (split.cu): a host batch of >= 1024 traces runs as two
# halves on two threads / streams, and stw_plan_batches as two lanes
if os.environ.get("STW_SAN_CONCURRENT"):
    big = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(1024)]
    bpa = api.plan_batch(big, tracegen.C4_CANDIDATES, select_best=True)
    os.environ["STW_NO_SPLIT"] = "1"
    bpb = api.plan_batch(big, tracegen.C4_CANDIDATES, select_best=True)
    del os.environ["STW_NO_SPLIT"]
    assert np.array_equal(bpa.addr, bpb.addr) and np.array_equal(bpa.stats, bpb.stats), "split call"
    many = api.plan_batches([tas[:16], tas[16:32], tas[32:]], tracegen.C4_CANDIDATES, select_best=True)
    for k, g in enumerate((tas[:16], tas[16:32], tas[32:])):
        w = api.plan_batch(g, tracegen.C4_CANDIDATES, select_best=True)
        assert np.array_equal(many[k].addr, w.addr) and np.array_equal(many[k].addr_best, w.addr_best), "two lanes"
print("sanitize workload ok")
