import sys; sys.path.insert(0, "/root/repo")
from paper_2507_16274_b200 import api, tracegen
ta = tracegen.synth_arrays(tracegen.config("c5_llama3_70b"))
api.plan_batch([ta], ((True, True),), detail=False)
