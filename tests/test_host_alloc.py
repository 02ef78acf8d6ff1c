"""The native allocator core (libstw_alloc.so: stw_cache_*, stw_reuse_best_fit)
behind the reference's `CachingAllocator` and `dynamic_allocate`. Host code,
so these run on CPU. Known answers from the reference's tests
(pkg/tests/test_baseline.py:15-107, test_sim.py:55-80), random op sequences
against oracle/subops.py."""

import random

import pytest

from oracle import subops as O
from paper_2507_16274_b200.baseline import MIN_SEGMENT, CachingAllocator
from paper_2507_16274_b200.domain import SimulationError
from paper_2507_16274_b200.ivset import Interval, IntervalSet
from paper_2507_16274_b200.sim import PoolState, dynamic_allocate

U = 512
MIB = 1 << 20


def test_split_and_merge_round_trip():
    c = CachingAllocator(min_segment=1024)
    assert (c.malloc(1, 512)[0], c.malloc(2, 512)[0]) == (0, 512)
    c.free(1)
    c.free(2)
    assert c.segments[0].free == [(0, 1024)]


def test_best_fit_prefers_tightest_block():
    c = CachingAllocator(min_segment=512)
    c.malloc(1, 4096)
    c.malloc(2, 1024)
    c.free(1)
    c.free(2)
    assert c.malloc(3, 1024) == (4096, 0)


def test_interleaved_pattern_reserves_ten_mib():
    """test_baseline.py:25-46 hand-replayed: 4 MiB, 2 MiB, free, 2 MiB split, 4 MiB miss."""
    c = CachingAllocator()
    assert c.malloc(1, 4 * MIB) == (0, 4 * MIB)
    assert c.malloc(2, 2 * MIB) == (4 * MIB, 2 * MIB)
    c.free(1)
    assert c.malloc(3, 2 * MIB) == (0, 0)
    assert c.malloc(4, 4 * MIB) == (6 * MIB, 4 * MIB)
    assert c.reserved == 10 * MIB and c.live_bytes == 8 * MIB
    assert [s.end for s in c.segments] == [4 * MIB, 6 * MIB, 10 * MIB]


def test_errors():
    c = CachingAllocator()
    with pytest.raises(SimulationError, match="unknown id"):
        c.free(7)
    c.malloc(1, 512)
    assert c.owns(1) and not c.owns(2)
    with pytest.raises(SimulationError, match="already live"):
        c.malloc(1, 512)


def test_base_offset_and_default_segment():
    c = CachingAllocator(base=12345 * U)
    assert c.malloc(0, 3 * MIB) == (12345 * U, 4 * MIB)
    assert MIN_SEGMENT == 2 * MIB


def test_random_sequences_vs_oracle():
    rng = random.Random(1)
    for trial in range(30):
        base = rng.choice([0, 7 * U])
        mins = rng.choice([512, 4096, MIN_SEGMENT])
        c, o = CachingAllocator(base=base, min_segment=mins), O.Cache(base, mins)
        live = []
        for rid in range(400):
            if live and rng.random() < 0.45:
                r = live.pop(rng.randrange(len(live)))
                assert c.free(r) == o.free(r)
            else:
                size = rng.randint(1, 64) * U
                assert c.malloc(rid, size) == o.malloc(rid, size), (trial, rid)
                live.append(rid)
            assert c.reserved == o.reserved
        assert [(s.base, s.size, s.free) for s in c.segments] == [(g[0], g[1], g[2]) for g in o.segs]


def test_dynamic_allocate_candidate_selection():
    state = PoolState(100 * U, IntervalSet([Interval(0, 50 * U), Interval(80 * U, 100 * U)]), {})
    spaces = {("a", "b"): IntervalSet([Interval(30 * U, 90 * U)])}
    assert dynamic_allocate(state, spaces, ("a", "b"), 16 * U) == 30 * U
    assert not state.free.contains_interval(Interval(30 * U, 46 * U))
    assert state.free.contains_interval(Interval(46 * U, 50 * U))


def test_dynamic_allocate_fallbacks():
    state = PoolState.fresh(100 * U)
    assert dynamic_allocate(state, {("a", "b"): IntervalSet.empty()}, ("a", "b"), U) is None
    assert dynamic_allocate(state, {}, ("missing", "key"), U) is None
    small = PoolState.fresh(10 * U)
    assert dynamic_allocate(small, {("a", "b"): IntervalSet.span(0, 10 * U)}, ("a", "b"), 11 * U) is None


def test_dynamic_allocate_random_vs_oracle():
    rng = random.Random(4)
    for _ in range(300):
        def rand_set():
            pts = sorted(rng.sample(range(0, 200), 2 * rng.randint(0, 6)))
            return IntervalSet([Interval(pts[i] * U, pts[i + 1] * U) for i in range(0, len(pts), 2)])

        free, space = rand_set(), rand_set()
        size = rng.randint(1, 40) * U
        want = O.reuse_best_fit([(iv.lo, iv.hi) for iv in free], [(iv.lo, iv.hi) for iv in space], size)
        state = PoolState(200 * U, free, {})
        assert dynamic_allocate(state, {"k": space}, "k", size) == want
        if want is not None:
            assert state.free == free.remove(Interval(want, want + size))
