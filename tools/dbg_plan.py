import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2507_16274_b200 import api, tracegen
from oracle import oracle as O
sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/tools")
from test_gpu_plan import fuzz_cfg, CANDS, STAT_MAP
def run(tas, cands=CANDS, verbose=True):
    bp = api.plan_batch(tas, cands)
    nbad = 0
    for t, ta in enumerate(tas):
        s0, s1 = int(bp.batch.ev_off[t]), int(bp.batch.ev_off[t + 1])
        for c, (f, g) in enumerate(cands):
            ref = O.plan(ta, f, g); u = t * len(cands) + c
            stat = ~ta.dyn.astype(bool)
            got = bp.addr[c, s0:s1]
            bad = np.nonzero((got != ref.addr) & stat)[0]
            sdiff = {n: (int(bp.stats[u, k]), ref.stats[n]) for k, n in enumerate(STAT_MAP) if int(bp.stats[u, k]) != ref.stats[n]}
            if bad.size or sdiff or bp.rc[u]:
                nbad += 1
                if verbose and nbad < 6:
                    print("trace", t, "cand", c, "rc", bp.rc[u], "bad", bad[:8].tolist(), "statdiff", sdiff)
                    print("   got layer", bp.layer_of[c, s0:s1][bad[:8]].tolist(), "ref layer", ref.layer_of[bad[:8]].tolist())
    print("units", len(tas) * len(cands), "bad", nbad)
tas = [tracegen.synth_arrays(fuzz_cfg(s)) for s in range(40)]
print("single trace 0:"); run(tas[:1])
print("single trace 0, cand TT only:"); run(tas[:1], ((True, True),))
print("single trace 0, cand FT only:"); run(tas[:1], ((False, True),))
print("batch 40:"); run(tas)
