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
