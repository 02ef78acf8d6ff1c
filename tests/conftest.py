"""Shared fixtures. `-m gpu` tests need a B200; everything else runs on CPU.

The reference package (/root/reference) is only present in the build
container: tests that run it live are skipped elsewhere, and the committed
fixtures under tests/golden/ (made by tests/golden/make_golden.py from the
reference) carry the pinning to the GPU box.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(os.path.join(REF_SRC, "memplan"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libstw.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def ref():
    """Import the reference memplan package (read-only path) or skip."""
    if not HAVE_REF:
        pytest.skip("reference package not present on this machine")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import memplan

    return memplan


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch.device("cuda:0")
