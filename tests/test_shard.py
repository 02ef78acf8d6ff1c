"""One large trace over several ranks: the band/halo split of
K7, the clipped time bands of K1 and the dealt keys of K8 reproduce the
single-process results. CPU tests check the decomposition with the oracle as
the per-band worker (and over gloo, world_size 2); the GPU tests run it on the
device kernels."""

import os
import socket

import numpy as np
import pytest

from paper_2507_16274_b200 import shard
from paper_2507_16274_b200.plan_types import DecisionColumns


def _rand_plan(seed, n=400, span=60, conflicts=True):
    """Random rectangles; with `conflicts`, addresses collide often (ties included)."""
    rng = np.random.default_rng(seed)
    ts = rng.integers(0, span, n)
    te = ts + rng.integers(1, 12, n)
    size = rng.integers(1, 5, n) * 512
    if conflicts:
        addr = rng.integers(0, 40, n) * 512
    else:  # one layer per rectangle: never overlaps
        addr = np.arange(n, dtype=np.int64) * 8 * 512
    ids = rng.permutation(n * 3)[:n]
    return DecisionColumns(ids, addr, size, ts, te)


def _oracle_validate(*cols):
    from oracle import oracle as O

    n, pairs = O.validate(*cols)
    assert n == len(pairs)
    return pairs


def _full(cols):
    return _oracle_validate(cols.id, cols.addr, cols.size, cols.t_s, cols.t_e)


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_validate_bands_concatenate_to_the_full_report(seed, world):
    cols = _rand_plan(seed)
    want = _full(cols)
    assert len(want) > 0
    got = np.concatenate([shard.validate_band(cols, r, world, _oracle_validate) for r in range(world)])
    assert got.tolist() == want.tolist()


def test_validate_bands_valid_plan_and_tiny_world_split():
    cols = _rand_plan(3, n=50, conflicts=False)
    assert len(_full(cols)) == 0
    for world in (1, 4, 64):  # more ranks than decisions: empty bands
        assert sum(len(shard.validate_band(cols, r, world, _oracle_validate)) for r in range(world)) == 0


@pytest.mark.parametrize("world", [1, 2, 3, 7])
def test_peak_bands_max_is_the_peak(world):
    from oracle import oracle as O

    for seed in range(3):
        c = _rand_plan(seed, n=300)
        want = O.peak_live(c.size, c.t_s, c.t_e)
        got = max(shard.peak_band(c.size, c.t_s, c.t_e, r, world, O.peak_live) for r in range(world))
        assert got == want


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cols = _rand_plan(7)
        rows = np.concatenate(shard.allgather_rows(shard.validate_band(cols, rank, world, _oracle_validate)))
        pk = shard._allreduce_max(shard.peak_band(cols.size, cols.t_s, cols.t_e, rank, world, O.peak_live))
        q.put((rank, rows.tolist(), pk))
    finally:
        dist.destroy_process_group()


def test_sharded_validate_and_peak_over_gloo():
    import torch.multiprocessing as mp

    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    cols = _rand_plan(7)
    want = _full(cols).tolist()
    peak = O.peak_live(cols.size, cols.t_s, cols.t_e)
    for _, rows, pk in res:
        assert rows == want
        assert pk == peak


# ---------------------------------------------------------------- device
@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_device_validate_bands_match_full_device_report(world):
    from paper_2507_16274_b200 import api

    for seed in range(3):
        cols = _rand_plan(seed, n=3000, span=400)
        want = api.validate_columns(cols.id, cols.addr, cols.size, cols.t_s, cols.t_e)
        assert want.tolist() == _full(cols).tolist()
        got = np.concatenate([shard.validate_band(cols, r, world) for r in range(world)])
        assert got.tolist() == want.tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 8])
def test_device_peak_bands_and_planned_c1(world):
    from oracle import oracle as O
    from paper_2507_16274_b200 import api, tracegen

    c = _rand_plan(5, n=5000, span=2000)
    want = O.peak_live(c.size, c.t_s, c.t_e)
    assert max(shard.peak_band(c.size, c.t_s, c.t_e, r, world) for r in range(world)) == want
    # a real planned trace: bands of its valid plan report nothing; peaks agree
    tr = tracegen.synth_trace(tracegen.config("c1_llama2_7b_1f1b"))
    plan = api.synthesize_static_plan(tr)
    cols = plan.columns()
    assert sum(len(shard.validate_band(cols, r, world)) for r in range(world)) == 0
    assert max(shard.peak_band(cols.size, cols.t_s, cols.t_e, r, world) for r in range(world)) == \
        api.peak_live_bytes(tr.static_events())


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_device_reuse_keys_dealt_over_ranks(world):
    from paper_2507_16274_b200 import api, tracegen

    tr = tracegen.synth_trace(tracegen.config("c3_mixtral_moe"))
    plan = api.synthesize_static_plan(tr)
    want = api.derive_reuse_map(plan, tr)
    parts = [shard.reuse_rows(plan, tr, r, world) for r in range(world)]
    keys, t_lo, t_hi, _ = parts[0]
    assert len(keys) > 1
    got = shard.assemble_reuse_map(keys, t_lo, t_hi, np.concatenate([p[3] for p in parts]))
    assert got == want
