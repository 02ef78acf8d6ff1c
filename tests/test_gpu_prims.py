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


def test_radix_sort_full_bench_size_properties(cuda):
    """The bench's K2 size (2^27 pairs, 42 key bits, >> L2), checked on the
    device by size-independent properties: keys nondecreasing, values a
    permutation, and values increasing inside runs of equal keys (stable)."""
    import torch

    n, bits = 1 << 27, 42
    g = torch.Generator(device=cuda).manual_seed(3)
    k = torch.randint(0, 1 << bits, (n,), generator=g, device=cuda, dtype=torch.int64)
    k[::5] = k[1]  # long runs of one key
    v = torch.arange(n, dtype=torch.int32, device=cuda)
    api.radix_sort_pairs(k, v, 0, bits)
    assert bool((k[1:] >= k[:-1]).all())
    same = k[1:] == k[:-1]
    assert bool((v[1:][same] > v[:-1][same]).all())
    seen = torch.zeros(n, dtype=torch.bool, device=cuda)
    seen[v.long()] = True
    assert bool(seen.all())


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


def _c4_rect_sets(n_traces, cuda):
    """Sweep-ordered static rectangles of the c4 plans (4 candidates) on the device."""
    import torch

    tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(n_traces)]
    bp = api.plan_batch(tas, tracegen.C4_CANDIDATES)
    off, ts, te, sz, ad = [0], [], [], [], []
    for t, ta in enumerate(tas):
        s0 = int(bp.batch.ev_off[t])
        o = np.lexsort((ta.id, ta.t_s))  # sweep order (t_s, id)
        o = o[ta.dyn[o] == 0]
        ts.append(ta.t_s[o])
        te.append(ta.t_e[o])
        sz.append(ta.size[o])
        ad.append(bp.addr[:, s0 + o])
        off.append(off[-1] + o.size)
    cat = lambda xs, dt: torch.from_numpy(np.ascontiguousarray(np.concatenate(xs, axis=-1), dtype=dt)).to(cuda)  # noqa
    return (torch.tensor(off, dtype=torch.int64, device=cuda), cat(ts, np.int32), cat(te, np.int32),
            cat(sz, np.int64), cat(ad, np.int64))


def test_validate_sets_valid_and_conflicting(cuda):
    """Batched K7 (fast overlap sweep + exact fallback) vs the oracle's validate_plan."""
    off, ts, te, sz, ad = _c4_rect_sets(48, cuda)
    assert int(api.validate_sets(off, ts, te, sz, ad).abs().sum()) == 0
    rng = np.random.default_rng(7)
    h_ad = ad.cpu().numpy().copy()
    h_off, h_ts, h_te, h_sz = off.cpu().numpy(), ts.cpu().numpy(), te.cpu().numpy(), sz.cpu().numpy()
    for _ in range(40):  # move random rectangles onto other addresses (conflicts in most units)
        c, k = int(rng.integers(0, 4)), int(rng.integers(0, h_ts.size))
        h_ad[c, k] = h_ad[c, int(rng.integers(0, h_ts.size))]
    h_ad[1, 5] += 256  # not a multiple of 2^9: that unit takes the exact reporter
    import torch

    got = api.validate_sets(off, ts, te, sz, torch.from_numpy(h_ad).to(cuda)).cpu().numpy()
    for s in range(h_off.size - 1):
        a, b = h_off[s], h_off[s + 1]
        for c in range(4):
            ids = np.arange(b - a, dtype=np.int64)
            n_ref, _ = O.validate(ids, h_ad[c, a:b], h_sz[a:b], h_ts[a:b], h_te[a:b])
            assert got[s * 4 + c] == n_ref, (s, c)
