"""Live training under the plan (tools/matcher_demo.py, fresh process): the
Allocation Profiler records a small MoE model's iteration through the Request
Matcher's hooks, the device plans it, and the next iteration -- served by
libstw_alloc as PyTorch's CUDA allocator -- lands every request where
simulate's log says (same route, same replay address), with the replay's
metrics and unchanged model results."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_live_model_served_from_its_own_plan():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "matcher_demo.py")], capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    out = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert out["dynamic"] > 0 and out["routes"]["planned"] > 0
    assert out["same_address_stream"], out
    assert out["same_metrics"] and out["same_losses"], out
