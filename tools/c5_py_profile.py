import sys, time
sys.path.insert(0, "/root/repo")
import paper_2507_16274_b200 as M
from paper_2507_16274_b200 import tracegen, api
from paper_2507_16274_b200.batching import HostBatch
tr = M.Trace.from_arrays(tracegen.synth_arrays(tracegen.config("c5_llama3_70b")))
M.synthesize_static_plan(tr)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(3): M.synthesize_static_plan(tr)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
