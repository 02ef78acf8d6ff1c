"""K1 (peak live bytes) and K2 (radix sort) on the device vs the oracle / numpy."""

import numpy as np
import pytest

from paper_2507_16274_b200 import api, soa, tracegen
from paper_2507_16274_b200.batching import HostBatch
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,bits", [(1, 8), (1000, 13), (4095, 64), (4097, 20), (1_000_003, 42), (3_000_000, 64)])
def test_radix_sort_stable_matches_numpy(cuda, n, bits):
    import torch

    rng = np.random.default_rng(n)
    keys = rng.integers(0, 2**63 - 1, size=n, dtype=np.int64)
    if bits < 64:
        keys &= (1 << bits) - 1
    keys[::7] = keys[0]  # duplicates exercise stability
    vals = np.arange(n, dtype=np.int32)
    k = torch.from_numpy(keys).to(cuda)
    v = torch.from_numpy(vals).to(cuda)
    api.radix_sort_pairs(k, v, 0, bits)
    order = np.argsort(keys.view(np.uint64), kind="stable")
    assert np.array_equal(v.cpu().numpy(), order.astype(np.int32))
    assert np.array_equal(k.cpu().numpy(), keys[order])


def test_radix_sort_partial_bits(cuda):
    import torch

    rng = np.random.default_rng(1)
    keys = rng.integers(0, 1 << 40, size=50_000, dtype=np.int64)
    k = torch.from_numpy(keys).to(cuda)
    v = torch.arange(keys.size, dtype=torch.int32, device=cuda)
    api.radix_sort_pairs(k, v, 16, 32)  # sort on bits [16, 32) only
    order = np.argsort((keys >> 16) & 0xFFFF, kind="stable")
    assert np.array_equal(v.cpu().numpy(), order.astype(np.int32))


def _peak_oracle(ta, static_only=False):
    m = ta.dyn == 0 if static_only else np.ones(len(ta), bool)
    return O.peak_live(ta.size[m], ta.t_s[m], ta.t_e[m])


@pytest.mark.parametrize("name", list(tracegen.CONFIGS))
def test_peak_live_configs(cuda, name):
    ta = tracegen.synth_arrays(tracegen.config(name))
    assert api.peak_live_bytes(ta) == _peak_oracle(ta)


def test_peak_live_fuzz_and_edges(cuda):
    from paper_2507_16274_b200.domain import MemoryRequestEvent, PhaseId

    F, B = PhaseId.parse("F:0"), PhaseId.parse("B:0")
    # model tests: test_model.py:72-82
    a = MemoryRequestEvent(0, 10 * 512, 0, 5, F, B)
    b = MemoryRequestEvent(1, 20 * 512, 2, 8, F, B)
    assert api.peak_live_bytes([a, b]) == 30 * 512
    assert api.peak_live_bytes([MemoryRequestEvent(2, 7 * 512, 0, 3, F, B)]) == 7 * 512
    c = MemoryRequestEvent(3, 10 * 512, 0, 4, F, B)
    d = MemoryRequestEvent(4, 20 * 512, 4, 9, F, B)
    assert api.peak_live_bytes([c, d]) == 20 * 512  # touching lifespans
    assert api.peak_live_bytes([]) == 0
    rng = np.random.default_rng(0)
    for it in range(30):
        n = int(rng.integers(1, 300))
        ts = rng.integers(0, 1000, n)
        te = ts + rng.integers(1, 200, n)
        evs = [MemoryRequestEvent(i, 512 * int(rng.integers(1, 50)), int(ts[i]), int(te[i]), F, B) for i in range(n)]
        ta = soa.from_events(evs)
        assert api.peak_live_bytes(evs) == _peak_oracle(ta)


def test_peak_live_batched(cuda):
    import ctypes as C

    from paper_2507_16274_b200 import _lib

    tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(64)]
    hb = HostBatch(tas)
    out = np.zeros(len(tas), np.int64)
    err = _lib.errbuf()
    b = hb.struct()
    _lib.check(_lib.load().stw_peak_live(C.byref(b), 1, _lib.ptr(out), None, err, 1024), err)
    assert out.tolist() == [_peak_oracle(t, static_only=True) for t in tas]
