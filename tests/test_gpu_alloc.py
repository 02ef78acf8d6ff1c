"""The runtime allocator (libstw_alloc.so): its address stream
equals simulate's log on the same trace and plan, and it works as PyTorch's
CUDAPluggableAllocator."""

import os
import subprocess
import sys

import pytest

import paper_2507_16274_b200 as M
from paper_2507_16274_b200 import tracegen
from paper_2507_16274_b200.runtime import PlanAllocator

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def check(ta):
    tr = M.Trace.from_arrays(ta)
    plan, rmap = M.plan_trace(tr)
    bundle = plan.to_bundle(rmap)
    rep, log = M.simulate(tr, bundle)
    want = [(r["id"], r["route"], r["addr"]) for r in log if r["kind"] == "alloc"]
    rt = PlanAllocator(bundle, tr)
    try:
        got = rt.replay()
        assert got == want
        assert rt.report() == rep  # same metrics as the replay scorer
    finally:
        rt.shutdown()


@pytest.mark.parametrize("preset,seed", [("dense", 0), ("moe", 2), ("moe_recompute", 1), ("dense_vpp_recompute", 3)])
def test_allocator_matches_replay_presets(preset, seed):
    check(tracegen.synth_arrays(tracegen.SynthConfig.for_preset(preset, seed=seed)))


@pytest.mark.parametrize("name", ["c1_llama2_7b_1f1b", "c3_mixtral_moe", "c3b_mixtral_moe_rcp"])
def test_allocator_matches_replay_configs(name):
    check(tracegen.synth_arrays(tracegen.config(name)))


def test_allocator_as_torch_pluggable_allocator():
    """Fresh process: install before any CUDA allocation, allocate tensors under the plan."""
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "alloc_torch_demo.py")], capture_output=True,
                         text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "torch pluggable allocator ok" in res.stdout
