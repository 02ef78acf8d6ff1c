"""Planner parity: libstw (stw_plan_batch) vs the C oracle, bit-exact.

Addresses of every static event, pool size, every PlanStats counter, the
accepted-fusion audit pairs (exact doubles) and the layer table, under all
four (fusion, gap_insert) candidates."""

import numpy as np
import pytest

from paper_2507_16274_b200 import api, tracegen
from paper_2507_16274_b200.batching import HostBatch
from oracle import oracle as O

pytestmark = pytest.mark.gpu

CANDS = tracegen.C4_CANDIDATES
STAT_MAP = ("num_events", "num_persistent", "num_groups", "num_plans", "num_residuals", "fusion_attempts",
            "fusion_accepted", "gap_insertions", "num_layers", "pool_size", "static_peak", "persistent_size")


def fuzz_cfg(seed):
    preset = tracegen.PRESETS[seed % 6]
    return tracegen.SynthConfig.for_preset(preset, seed=seed, num_layers=4 + seed % 9,
                                          num_microbatches=1 + seed % 4, transient_ratio=0.2 + (seed % 5) * 0.2)


def check_batch(tas, cands=CANDS):
    bp = api.plan_batch(tas, cands)
    C = len(cands)
    for t, ta in enumerate(tas):
        s0, s1 = int(bp.batch.ev_off[t]), int(bp.batch.ev_off[t + 1])
        for c, (f, g) in enumerate(cands):
            ref = O.plan(ta, f, g)
            u = t * C + c
            assert ref.rc == 0 and bp.rc[u] == 0, (t, c, ref.err, bp.rc[u])
            stat = ~ta.dyn.astype(bool)
            got = bp.addr[c, s0:s1]
            bad = np.nonzero(got[stat] != ref.addr[stat])[0]
            assert bad.size == 0, (t, c, "addr mismatch", bad[:5], got[stat][bad[:5]], ref.addr[stat][bad[:5]])
            for k, name in enumerate(STAT_MAP):
                assert int(bp.stats[u, k]) == ref.stats[name], (t, c, name, int(bp.stats[u, k]), ref.stats[name])
            na = ref.stats["n_accepted"]
            assert bp.fus_tmp[c, s0:s0 + na].tolist() == [a for a, _ in ref.accepted]
            assert bp.fus_avg[c, s0:s0 + na].tolist() == [b for _, b in ref.accepted]
            nl = ref.stats["num_layers"]
            assert bp.layer_base[c, s0:s0 + nl].tolist() == ref.layer_base.tolist()
            assert bp.layer_size[c, s0:s0 + nl].tolist() == ref.layer_size.tolist()
            assert np.array_equal(bp.layer_of[c, s0:s1][stat], ref.layer_of[stat])
    return bp


def test_plan_fuzz_batched():
    tas = [tracegen.synth_arrays(fuzz_cfg(s)) for s in range(200)]
    check_batch(tas)


def test_plan_fuzz_single_calls():
    for s in range(0, 60, 7):
        check_batch([tracegen.synth_arrays(fuzz_cfg(s))])


def test_plan_c4_sample_batched():
    tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(0, 4096, 16)]
    bp = check_batch(tas)
    assert bp.rc.max() == 0


@pytest.mark.parametrize("name", ["c1_llama2_7b_1f1b", "c3_mixtral_moe", "c3b_mixtral_moe_rcp", "c2_llama2_7b_vpp_rcp"])
def test_plan_configs(name):
    check_batch([tracegen.synth_arrays(tracegen.config(name))], ((True, True),))


def test_plan_select_best():
    tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(32)]
    bp = api.plan_batch(tas, CANDS, select_best=True)
    for t, ta in enumerate(tas):
        pools = [O.plan(ta, f, g).stats["pool_size"] for f, g in CANDS]
        best = min(range(4), key=lambda c: (pools[c], c))
        assert int(bp.best_cand[t]) == best and int(bp.best_pool[t]) == pools[best]
        s0, s1 = int(bp.batch.ev_off[t]), int(bp.batch.ev_off[t + 1])
        assert np.array_equal(bp.addr_best[s0:s1], bp.addr[best, s0:s1])


def _manual_trace(specs, phases):
    """specs: (id, size_bytes, t_s, t_e, p_s, p_e); phases: [(tag, start, end)]"""
    from paper_2507_16274_b200 import soa
    from paper_2507_16274_b200.domain import MemoryRequestEvent, PhaseId, PhaseSpan

    evs = [MemoryRequestEvent(i, s, a, b, PhaseId.parse(x), PhaseId.parse(y)) for i, s, a, b, x, y in specs]
    sched = [PhaseSpan(PhaseId.parse(t), a, b) for t, a, b in phases]
    return soa.from_events(evs, sched)


def test_plan_many_layers_overflow_paths():
    rng = np.random.default_rng(7)
    tas = []
    # 150 simultaneously live same-size events (one class, 150 layers) + distinct sizes (150 classes)
    specs = [(i, 512 * 4, i, 400 + i, "F:0", "F:0") for i in range(150)]
    tas.append(_manual_trace(specs, [("F:0", 0, 1000)]))
    specs = [(i, 512 * (i + 1), i, 400 + i, "F:0", "F:0") for i in range(150)]
    tas.append(_manual_trace(specs, [("F:0", 0, 1000)]))
    # random single-phase soup with a few hundred layers worth of overlap
    specs = []
    for i in range(3000):
        s = int(rng.integers(0, 2000))
        specs.append((i * 7 + 3, 512 * int(rng.integers(1, 6)), s, s + int(rng.integers(1, 600)), "F:0", "F:0"))
    tas.append(_manual_trace(specs, [("F:0", 0, 3000)]))
    check_batch(tas)
    check_batch(tas[2:])
    # without gap insertion every narrow unit runs in the zero-smem launch: its
    # > 32-layer units must still reach the CTA kernel
    check_batch(tas, ((True, False), (False, False)))
    check_batch(tas[:1], ((False, False),))


def test_plan_batches_pipeline_matches_single_calls():
    """stw_plan_batches (double-buffered staging across batches) == stw_plan_batch per batch."""
    groups = [[tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(a, b)] for a, b in
              ((0, 40), (40, 47), (100, 164), (7, 8))]
    many = api.plan_batches(groups, tracegen.C4_CANDIDATES, select_best=True)
    for g, got in zip(groups, many):
        want = api.plan_batch(g, tracegen.C4_CANDIDATES, select_best=True)
        for f in ("rc", "err_ids", "stats", "addr", "layer_of", "layer_base", "layer_size", "order", "best_cand",
                  "best_pool", "addr_best"):
            assert np.array_equal(getattr(got, f), getattr(want, f)), f
        assert np.array_equal(got.fus_tmp.view(np.int64), want.fus_tmp.view(np.int64))


def test_plan_batches_compact_upload():
    """Host batches with compact columns (HostBatch.pack: int32 id offsets,
    sizes in power-of-two units, widened on the device) plan exactly like the
    full-width upload; mixed packed / unpacked batches in one call."""
    from paper_2507_16274_b200.batching import HostBatch

    groups = [[tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(a, b)] for a, b in
              ((0, 24), (24, 31), (50, 90))]
    hbs = [HostBatch(g, pinned=True) for g in groups]
    assert hbs[0].pack() and hbs[2].pack()
    assert hbs[0].upload_nbytes < hbs[0].nbytes
    many = api.plan_batches(hbs, tracegen.C4_CANDIDATES, select_best=True)
    for g, got in zip(groups, many):
        want = api.plan_batch(g, tracegen.C4_CANDIDATES, select_best=True)
        for f in ("rc", "stats", "addr", "best_cand", "best_pool", "addr_best"):
            assert np.array_equal(getattr(got, f), getattr(want, f)), f
    one = api.plan_batch(hbs[2], tracegen.C4_CANDIDATES, select_best=True)  # the single call stages compact too
    want = api.plan_batch(groups[2], tracegen.C4_CANDIDATES, select_best=True)
    for f in ("rc", "stats", "addr", "best_cand", "best_pool", "addr_best"):
        assert np.array_equal(getattr(one, f), getattr(want, f)), f


def test_plan_invariant_to_event_listing_order():
    """Shuffled event listings take the sorting path of the canonical ranks (the
    recorded order takes the identity fast path); plans must match by id."""
    import dataclasses

    rng = np.random.default_rng(5)
    tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(0, 96, 3)]
    shuf = []
    for ta in tas:
        p = rng.permutation(len(ta))
        shuf.append(dataclasses.replace(ta, **{k: getattr(ta, k)[p] for k in
                                               ("id", "size", "t_s", "t_e", "ps", "pe", "dyn", "ls", "le")}))
    a = api.plan_batch(tas, tracegen.C4_CANDIDATES, select_best=True)
    b = api.plan_batch(shuf, tracegen.C4_CANDIDATES, select_best=True)
    assert np.array_equal(a.stats, b.stats) and np.array_equal(a.best_cand, b.best_cand)
    for t, (ta, tb) in enumerate(zip(tas, shuf)):
        sa, sb = int(a.batch.ev_off[t]), int(b.batch.ev_off[t])
        n = len(ta)
        for c in range(4):
            ma = dict(zip(ta.id.tolist(), a.addr[c, sa:sa + n].tolist()))
            mb = dict(zip(tb.id.tolist(), b.addr[c, sb:sb + n].tolist()))
            assert ma == mb, (t, c)


@pytest.mark.parametrize("cands", [((True, True),), ((False, True),), ((True, False),), ((False, False),),
                                   ((False, True), (True, False)), CANDS])
def test_plan_edge_traces_and_candidate_subsets(cands):
    """Empty, single-event, persistent-only and cross-phase-only traces mixed into
    one batch with regular ones, under every candidate subset (each subset takes
    different launch paths: fusion on/off, gap/zero-smem layer launches)."""
    tas = [_manual_trace([], [("F:0", 0, 10)]),
           _manual_trace([(5, 1024, 2, 3, "F:0", "F:0")], [("F:0", 0, 10)]),
           _manual_trace([(i, 512 * (1 + i % 3), i, 40, "F:0", "B:0") for i in range(20)],
                         [("F:0", 0, 20), ("B:0", 20, 40)]),
           _manual_trace([(i, 512 * (1 + i % 2), i, 25 + i, "F:0", "B:0") for i in range(12)],
                         [("F:0", 0, 20), ("B:0", 20, 40)])]
    tas += [tracegen.synth_arrays(fuzz_cfg(s)) for s in (3, 11)]
    tas.insert(3, _manual_trace([], [("F:0", 0, 4)]))
    check_batch(tas, cands)


def test_plan_batches_with_empty_and_tiny_batches():
    """The pipelined call over batches of all-empty traces, one event, and a
    regular batch gives each batch's single-call result."""
    groups = [[_manual_trace([], [("F:0", 0, 10)]), _manual_trace([], [("F:0", 0, 3)])],
              [_manual_trace([(5, 1024, 2, 3, "F:0", "F:0")], [("F:0", 0, 10)])],
              [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(3)],
              [_manual_trace([], [("F:0", 0, 10)])]]
    many = api.plan_batches(groups, CANDS, select_best=True)
    for g, got in zip(groups, many):
        want = api.plan_batch(g, CANDS, select_best=True)
        for f in ("rc", "stats", "addr", "best_cand", "best_pool", "addr_best"):
            assert np.array_equal(getattr(got, f), getattr(want, f)), f


def test_failed_call_leaves_no_state_behind():
    """A call that fails midway (item sort key wider than 64 bits: one 2^61-byte
    event in a 4096-trace batch) raises, and the next call is still exact."""
    tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(4095)]
    tas.append(_manual_trace([(1, 1 << 61, 0, 2, "F:0", "F:0")], [("F:0", 0, 4)]))
    with pytest.raises(Exception, match="64 bits"):
        api.plan_batch(tas, CANDS)
    check_batch(tas[:8])


@pytest.mark.parametrize("on_device", [False, True])
def test_plan_split_call_matches_unsplit(on_device, monkeypatch):
    """Large host batches run as two concurrent halves (split.cu; device batches
    stay whole); every output field equals the unsplit call's (STW_NO_SPLIT),
    including the rebased event indices of erroring units in the second half,
    for host outputs and for device outputs of a host batch."""
    import ctypes as C

    import torch

    from paper_2507_16274_b200 import _lib

    tas = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(2048)]
    bad = _manual_trace([(1, 100, 0, 2, "F:0", "F:0"), (2, 512, 1, 3, "F:0", "F:0")], [("F:0", 0, 4)])
    tas[10] = bad
    tas[1900] = bad  # (the cut is near half of the events: both halves get one)
    hb = HostBatch(tas, pinned=True)
    T, N, Cn = hb.T, hb.N, len(CANDS)

    def run():
        if not on_device:
            return api.plan_batch(hb, CANDS, select_best=True)
        f = {"rc": (T * Cn, torch.int32), "err_ids": (2 * T * Cn, torch.int64), "stats": (T * Cn * _lib.NSTATS, torch.int64),
             "addr": (Cn * N, torch.int64), "layer_of": (Cn * N, torch.int32), "layer_base": (Cn * N, torch.int64),
             "layer_size": (Cn * N, torch.int64), "fus_tmp": (Cn * N, torch.float64), "fus_avg": (Cn * N, torch.float64),
             "order": (N, torch.int32), "best_cand": (T, torch.int32), "addr_best": (N, torch.int64),
             "best_pool": (T, torch.int64)}
        bufs = {k: torch.full((n,), -7, dtype=dt, device="cuda") for k, (n, dt) in f.items()}
        out = _lib.PlanOut(1, *[_lib.ptr(bufs[k]) for k in ("rc", "err_ids", "stats", "addr", "layer_of", "layer_base",
                                                             "layer_size", "fus_tmp", "fus_avg", "order", "best_cand",
                                                             "addr_best", "best_pool")])
        opts = _lib.PlanOpts(Cn, 1, _lib.ptr(api._cand_bits(CANDS)), 512, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        b = hb.struct()
        err = _lib.errbuf()
        _lib.check(_lib.load().stw_plan_batch(C.byref(b), C.byref(opts), C.byref(out), err, 1024), err)
        torch.cuda.synchronize()
        return {k: v.cpu().numpy() for k, v in bufs.items()}

    got = run()
    monkeypatch.setenv("STW_NO_SPLIT", "1")
    want = run()
    for k in ("rc", "err_ids", "stats", "addr", "layer_of", "layer_base", "layer_size", "fus_tmp", "fus_avg", "order",
              "best_cand", "addr_best", "best_pool"):
        a, b = (got[k], want[k]) if on_device else (getattr(got, k), getattr(want, k))
        if a.dtype == np.float64:
            a, b = a.view(np.int64), b.view(np.int64)
        assert np.array_equal(a, b), k
    rc = (got["rc"] if on_device else got.rc).reshape(T, Cn)
    err = (got["err_ids"] if on_device else got.err_ids).reshape(T, Cn, 2)
    assert (rc[10] != 0).all() and (rc[1900] != 0).all() and (rc[:10] == 0).all()
    assert (err[1900] >= 0).any() and int(err[1900].max()) >= int(hb.ev_off[1900])  # rebased into the batch


def test_plan_batches_two_lanes_error_in_second_lane():
    """stw_plan_batches runs even and odd batches in two concurrent lanes
    (split.cu); a batch failing in the worker's lane raises like the
    sequential pipeline, and the next call is exact."""
    good = [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(4095)]
    bad = good + [_manual_trace([(1, 1 << 61, 0, 2, "F:0", "F:0")], [("F:0", 0, 4)])]  # (as the test above)
    with pytest.raises(Exception, match="64 bits"):
        api.plan_batches([good[:4], bad, good[4:8]], CANDS, select_best=True)
    many = api.plan_batches([good[:4], good[4:8], good[8:]], CANDS, select_best=True)
    for g, got in zip((good[:4], good[4:8], good[8:]), many):
        want = api.plan_batch(g, CANDS, select_best=True)
        for f in ("rc", "stats", "addr", "best_cand", "best_pool", "addr_best"):
            assert np.array_equal(getattr(got, f), getattr(want, f)), f


def test_plan_batches_shared_outputs_keep_sequential_semantics():
    """Batches whose output structs share buffers run in one lane: the buffers
    end with the last batch's results, as with sequential calls."""
    import ctypes as C

    from paper_2507_16274_b200 import _lib

    groups = [[tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(a, a + 6)] for a in (0, 30, 60, 90)]
    hbs = [HostBatch(g, pinned=True) for g in groups]
    Cn = len(CANDS)
    maxU, maxN = max(h.T for h in hbs) * Cn, max(h.N for h in hbs)
    rc = np.full(maxU, -1, np.int32)
    stats = np.zeros(maxU * _lib.NSTATS, np.int64)
    abest = np.zeros(maxN, np.int64)
    bpool = np.zeros(max(h.T for h in hbs), np.int64)
    best = np.zeros(max(h.T for h in hbs), np.int32)
    out = _lib.PlanOut(0, _lib.ptr(rc), None, _lib.ptr(stats), None, None, None, None, None, None, None,
                       _lib.ptr(best), _lib.ptr(abest), _lib.ptr(bpool))
    opts = _lib.PlanOpts(Cn, 1, _lib.ptr(api._cand_bits(CANDS)), 512, None)
    bs = (_lib.Batch * 4)(*[h.struct() for h in hbs])
    outs = (_lib.PlanOut * 4)(*([out] * 4))
    err = _lib.errbuf()
    _lib.check(_lib.load().stw_plan_batches(4, bs, C.byref(opts), outs, err, 1024), err)
    want = api.plan_batch(groups[-1], CANDS, select_best=True)
    U, N = hbs[-1].T * Cn, hbs[-1].N
    assert np.array_equal(stats[:U * _lib.NSTATS].reshape(U, -1), want.stats)
    assert np.array_equal(abest[:N], want.addr_best) and np.array_equal(bpool[:hbs[-1].T], want.best_pool)
