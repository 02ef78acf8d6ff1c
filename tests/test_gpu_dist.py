"""bench.py's multi-rank sweep on ONE GPU: two ranks (gloo, both on cuda:0)
run the device planner through the same code as the NCCL run -- each plans its
block of the c4 traces, the per-step exchange (allreduce MIN of packed
(pool << 2 | cand), SUM of failing units) rebuilds the whole sweep's best
plans, and rank 0 checks them against the reference's c4 anchor."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_two_ranks_share_one_gpu(scaling):
    traces = "4096" if scaling == "strong" else "2048"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo", "--share-gpu",
           "--scaling", scaling, "--traces", traces, "--steps", "2", "--warmup", "1", "--no-cpu-baseline",
           "--no-kernel-sweep", "--no-configs"]
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    assert line["config"]["traces"] == (4096 if scaling == "strong" else 4096)
    assert line["config"]["traces_per_rank"] == (2048 if scaling == "strong" else 2048)
    assert line["verified"]["matches_reference"] and line["verified"]["failing_units"] == 0
