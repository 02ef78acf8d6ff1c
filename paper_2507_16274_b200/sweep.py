"""Multi-GPU batched sweep: shard (trace, candidate) units over
ranks, plan locally on each GPU, combine with one tiny collective.

Two layouts:
  * trace shards (default, weak scaling): rank r plans traces
    [r*T, (r+1)*T) under every candidate; the best plan of a trace is picked on
    the rank that owns it. The only exchange is the sweep summary
    (sum of best pools, violating units, planned allocations): one allreduce.
  * unit shards (strong scaling of one sweep): units u = t*C + c are dealt
    round-robin; each rank packs (pool_size << 2 | cand) per trace over the
    units it owns (INT64_MAX elsewhere) and an allreduce MIN over int64[T]
    yields argmin (pool, cand) -- ties to the lowest candidate, exactly the
    reference's tie-break -- on every rank.
The collectives go through torch.distributed (NCCL on the GPU box, gloo in
the CPU tests)."""

from __future__ import annotations

import numpy as np

INT64_MAX = np.iinfo(np.int64).max


def trace_shard(rank: int, world: int, per_rank: int) -> range:
    return range(rank * per_rank, (rank + 1) * per_rank)


def unit_shard(rank: int, world: int, n_traces: int, n_cand: int) -> np.ndarray:
    units = np.arange(n_traces * n_cand, dtype=np.int64)
    return units[units % world == rank]


def pack_best(pools: np.ndarray, rc: np.ndarray, units: np.ndarray, n_traces: int, n_cand: int) -> np.ndarray:
    """Per-trace min of (pool << 2 | cand) over the given units (INT64_MAX if none ok)."""
    if n_cand > 4:
        raise ValueError("packing reserves 2 bits for the candidate index")
    out = np.full(n_traces, INT64_MAX, dtype=np.int64)
    t = units // n_cand
    c = units % n_cand
    ok = rc == 0
    keys = (pools.astype(np.int64) << 2) | c
    np.minimum.at(out, t[ok], keys[ok])
    return out


def unpack_best(keys: np.ndarray):
    valid = keys != INT64_MAX
    return np.where(valid, keys >> 2, -1), np.where(valid, keys & 3, -1)


def allreduce(arr: np.ndarray, op: str, device=None) -> np.ndarray:
    """In-place style allreduce of a small int64/float64 vector via torch.distributed."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return arr
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op={"min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}[op])
    return t.cpu().numpy()


def combine_best(local_keys: np.ndarray, device=None):
    """Global argmin (pool, cand) per trace from every rank's packed keys."""
    return unpack_best(allreduce(local_keys, "min", device))


def combine_summary(best_pool_sum: int, bad_units: int, planned: int, device=None) -> np.ndarray:
    return allreduce(np.asarray([best_pool_sum, bad_units, planned], dtype=np.int64), "sum", device)
