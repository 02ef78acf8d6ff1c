"""The C-ABI boundary: libstw.so builds for sm_100a, loads without a GPU, and
exports exactly what include/stw.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stw.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(stw_\w+)\s*\(", text)))


def test_header_declares_the_reference_replacements():
    names = declared_functions()
    for must in ("stw_peak_live", "stw_radix_sort_pairs", "stw_plan_batch", "stw_validate", "stw_validate_sets",
                 "stw_reuse_map",
                 "stw_simulate", "stw_baseline", "stw_version"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2507_16274_b200 import _lib

    lib = _lib.load()  # builds in-tree if stale; loading needs no GPU
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (stw_\w+)", out))
    assert set(declared_functions()) <= exported


def _declared(header):
    text = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", header)).read(), flags=re.S)
    return sorted(set(re.findall(r"\b(stw_\w+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("stw_alloc.h", "libstw_alloc.so"), ("stw_io.h", "libstw_io.so")])
def test_host_libraries_export_their_headers(header, lib):
    """libstw_alloc.so (runtime allocator + CachingAllocator core) and
    libstw_io.so (trace/plan files) export every function their header
    declares and load without a GPU."""
    from paper_2507_16274_b200 import build, runtime, traceio

    build.build_alloc()
    build.build_io()
    path = os.path.join(ROOT, "paper_2507_16274_b200", lib)
    L = runtime.load() if lib == "libstw_alloc.so" else traceio.load()
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (stw_\w+)", out))
    names = set(_declared(header)) - set(declared_functions())
    assert names and names <= exported, names - exported
    for n in names:
        assert hasattr(L, n)


def test_sub_operations_declared():
    names = declared_functions()
    for must in ("stw_group_events", "stw_local_plans", "stw_weighted_tmp", "stw_fuse_plans", "stw_build_layers",
                 "stw_metrics", "stw_release_scratch"):
        assert must in names


def test_library_is_sm100a_only():
    from paper_2507_16274_b200 import _lib

    _lib.load()
    res = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if res.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", res.stdout))
    assert arches == {"100a"}, arches


def test_version_string():
    from paper_2507_16274_b200 import _lib

    assert _lib.load().stw_version().decode().endswith("sm_100a")


def test_calls_fail_loudly_without_a_device():
    """No CPU fallback: without a GPU the library reports STW_ECUDA."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2507_16274_b200 import api
    from paper_2507_16274_b200.domain import DeviceError, MemoryRequestEvent, PhaseId

    ev = MemoryRequestEvent(0, 512, 0, 1, PhaseId.parse("F:0"), PhaseId.parse("F:0"))
    with pytest.raises(DeviceError):
        api.peak_live_bytes([ev])


def test_oracle_library_loads():
    from oracle import oracle as O

    lib = O.lib()
    for name in ("or_plan", "or_validate", "or_reuse", "or_simulate", "or_baseline", "or_peak_live"):
        assert hasattr(lib, name)
