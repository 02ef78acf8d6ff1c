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


def test_one_reserved_range_and_misuse_reporting():
    """Every block (pool or fallback) sits at range base + its replay address;
    unknown / double frees are reported; no teardown under live blocks; a plan
    reload keeps live blocks."""
    import ctypes as C

    from paper_2507_16274_b200 import runtime as R

    ta = tracegen.synth_arrays(tracegen.SynthConfig.for_preset("moe", seed=2, num_layers=4, num_microbatches=2))
    tr = M.Trace.from_arrays(ta)
    plan, rmap = M.plan_trace(tr)
    bundle = plan.to_bundle(rmap)
    rt = PlanAllocator(bundle, tr)
    L = R.load()
    base = rt.status()["base"]
    try:
        L.stw_set_layer(C.c_int32(-1), C.c_int32(1))  # dynamic with no reuse entry -> fallback segment
        p = L.stw_malloc(C.c_size_t(3 << 20), 0, None)
        v, route = PlanAllocator.vaddr(p)
        assert route == "fallback" and v >= bundle.pool_size and p == base + v
        with pytest.raises(M.DeviceError):
            PlanAllocator.shutdown()  # a block is live
        PlanAllocator(bundle, tr)  # reload keeps the live block
        assert PlanAllocator.vaddr(p)[0] == v
        L.stw_free(C.c_void_p(p), C.c_size_t(0), 0, None)
        L.stw_free(C.c_void_p(p), C.c_size_t(0), 0, None)  # double free
        with pytest.raises(M.SimulationError, match="unknown or already freed"):
            PlanAllocator.report()
    finally:
        L.stw_set_layer(C.c_int32(-1), C.c_int32(0))
        PlanAllocator.shutdown()
