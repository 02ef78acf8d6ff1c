"""Multi-rank sweep logic on CPU (gloo, world_size 2): sharding + the combine
collectives give the same best plan per trace as one process."""

import os
import socket

import numpy as np
import pytest

from paper_2507_16274_b200 import sweep, tracegen

T, CANDS = 12, tracegen.C4_CANDIDATES


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _unit_pools(units):
    from oracle import oracle as O

    pools, rc = [], []
    for u in units.tolist():
        t, c = divmod(u, len(CANDS))
        r = O.plan(tracegen.synth_arrays(tracegen.c4_config(t)), *CANDS[c])
        pools.append(r.stats["pool_size"])
        rc.append(r.rc)
    return np.asarray(pools, np.int64), np.asarray(rc, np.int32)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        units = sweep.unit_shard(rank, world, T, len(CANDS))
        pools, rc = _unit_pools(units)
        keys = sweep.pack_best(pools, rc, units, T, len(CANDS))
        best_pool, best_cand = sweep.combine_best(keys)
        summ = sweep.combine_summary(int(pools.sum()), int((rc != 0).sum()), len(units))
        q.put((rank, best_pool.tolist(), best_cand.tolist(), summ.tolist(), list(sweep.trace_shard(rank, world, 5))))
    finally:
        dist.destroy_process_group()


def test_unit_sharded_sweep_matches_single_process():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    units = np.arange(T * len(CANDS))
    pools, rc = _unit_pools(units)
    want_pool, want_cand = sweep.unpack_best(sweep.pack_best(pools, rc, units, T, len(CANDS)))
    grid = pools.reshape(T, len(CANDS))
    for t in range(T):  # argmin (pool, cand) as in SURVEY e1
        c = min(range(len(CANDS)), key=lambda k: (grid[t, k], k))
        assert (want_pool[t], want_cand[t]) == (grid[t, c], c)
    for rank, bp, bc, summ, seeds in res:
        assert bp == want_pool.tolist() and bc == want_cand.tolist()
        assert summ == [int(pools.sum()), 0, T * len(CANDS)]
        assert seeds == list(range(rank * 5, rank * 5 + 5))


def test_pack_best_tie_breaks_to_lowest_candidate():
    units = np.arange(8)
    pools = np.asarray([5, 5, 7, 5, 9, 8, 8, 8], np.int64)
    rc = np.zeros(8, np.int32)
    rc[0] = 2  # an erroring unit never wins
    bp, bc = sweep.unpack_best(sweep.pack_best(pools, rc, units, 2, 4))
    assert bp.tolist() == [5, 8] and bc.tolist() == [1, 1]
