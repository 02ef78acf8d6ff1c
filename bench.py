#!/usr/bin/env python
"""Benchmark of the hot path: the batched planner sweep.

One step = plan 4096 reference-exact synthetic dense-model traces under the 4
(fusion, gap_insert) candidates, self-check every plan (static peak + the
rectangle sweep), and pick the best candidate per trace -- i.e. 16,384 calls of
the reference's synthesize_static_plan. Weak scaling: rank r plans its own 4096
traces (seeds r*4096 .. r*4096+4095; rank 0's batch is exactly c4).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl stw|reference]

`--impl reference` times the CPU parity oracle (a C port of the reference
planner, oracle/) on the same workload with every host thread; it is the
reference arm. The JSON line follows the driver contract.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "planned allocations/sec"
UNIT = "allocs/s"
CANDS = ((True, True), (True, False), (False, True), (False, False))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="stw", choices=["stw", "reference"])
    ap.add_argument("--traces", type=int, default=4096, help="traces per rank (c4: 4096)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-print", action="store_true", help="per-kernel table on stderr")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def make_traces(rank: int, n: int):
    from paper_2507_16274_b200 import tracegen

    return [tracegen.synth_arrays(tracegen.c4_config(s)) for s in range(rank * n, (rank + 1) * n)]


# ---------------------------------------------------------------------------
# CPU side (oracle port of the reference planner)

def cpu_sweep(traces, threads: int):
    """Plan every trace x candidate with the C oracle on `threads` host threads.
    Returns (seconds, planned allocations)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    O.lib()

    def work(ta):
        n = 0
        for f, g in CANDS:
            r = O.plan(ta, f, g)
            assert r.rc == 0, r.err
            n += r.stats["num_events"]
        return n

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        total = sum(ex.map(work, traces))
    return time.perf_counter() - t0, total


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    traces = make_traces(0, args.traces)
    for _ in range(args.warmup):
        cpu_sweep(traces[: max(1, len(traces) // 16)], threads)
    times, total = [], 0
    for _ in range(args.steps):
        dt, total = cpu_sweep(traces, threads)
        times.append(dt)
    t = sum(times)
    value = total * args.steps / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic: reference-exact c4 traces (seeds 0..4095) regenerated from seeds",
        "config": {"workload": "c4_batched_sweep", "traces": len(traces), "candidates": 4,
                   "planned_allocs_per_step": total},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"full c4 sweep ({len(traces)} traces x 4 candidates) per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# algorithmic bytes per launch; w = workload counts of one step
def algo_bytes(kernel: str, w: dict, launches_per_step: float) -> float:
    per_step = {
        # planner layers: 32 B/event in + 8 B/event out, per unit (K5/K6)
        "k_layers": 40.0 * w["unit_events"],
        "k_layers_warp": 40.0 * w["unit_events"],
        # K2 radix passes: read+write (8 B key + 4 B value) per record per pass
        "k_radix_scatter": 24.0 * w["sort_records"],
        "k_radix_hist": 8.0 * w["sort_records"],
        # K7: 24 B per rectangle per candidate
        "k_validate_tiles": 24.0 * w["unit_events"],
        # fusion: the trace's events are read once per attempt at least
        "k_fusion": 32.0 * w["events"],
        # K1 timeline: 16 B/event read + 16 B/timestep
        "k_timeline_scatter": 16.0 * w["events"],
        "k_emit": 40.0 * w["unit_events"],
    }.get(kernel)
    if per_step is None:
        return float("nan")
    return per_step / max(launches_per_step, 1.0)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist

            # no collective is needed: rank 0 alone runs the CPU reference
            pass
        run_reference(args, rank, world)
        return

    import torch

    from paper_2507_16274_b200 import _lib, api
    from paper_2507_16274_b200.batching import HostBatch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    L = _lib.load()

    t_gen = time.perf_counter()
    traces = make_traces(rank, args.traces)
    t_gen = time.perf_counter() - t_gen
    hb = HostBatch(traces, pinned=True)
    db = hb.to_device(dev)
    T, N = hb.T, hb.N
    Cn = len(CANDS)
    cb = api._cand_bits(CANDS)
    stream = torch.cuda.current_stream(dev)
    sh = C.c_void_p(stream.cuda_stream)

    # device-resident outputs
    o_rc = torch.empty(T * Cn, dtype=torch.int32, device=dev)
    o_err = torch.empty(2 * T * Cn, dtype=torch.int64, device=dev)
    o_stats = torch.empty(T * Cn * _lib.NSTATS, dtype=torch.int64, device=dev)
    o_best = torch.empty(T, dtype=torch.int32, device=dev)
    o_bpool = torch.empty(T, dtype=torch.int64, device=dev)
    o_abest = torch.empty(N, dtype=torch.int64, device=dev)
    dev_out = _lib.PlanOut(1, _lib.ptr(o_rc), _lib.ptr(o_err), _lib.ptr(o_stats), None, None, None, None, None,
                           None, None, _lib.ptr(o_best), _lib.ptr(o_abest), _lib.ptr(o_bpool))
    opts = _lib.PlanOpts(Cn, 1, _lib.ptr(cb), 512, sh)
    dstruct = db.struct()
    err = _lib.errbuf()

    def step_device():
        _lib.check(L.stw_plan_batch(C.byref(dstruct), C.byref(opts), C.byref(dev_out), err, 1024), err)

    # host-side buffers for the end-to-end path (pinned in, pinned out)
    h_rc = torch.empty(T * Cn, dtype=torch.int32).pin_memory()
    h_err = torch.empty(2 * T * Cn, dtype=torch.int64).pin_memory()
    h_stats = torch.empty(T * Cn * _lib.NSTATS, dtype=torch.int64).pin_memory()
    h_best = torch.empty(T, dtype=torch.int32).pin_memory()
    h_bpool = torch.empty(T, dtype=torch.int64).pin_memory()
    h_abest = torch.empty(N, dtype=torch.int64).pin_memory()
    host_out = _lib.PlanOut(0, _lib.ptr(h_rc), _lib.ptr(h_err), _lib.ptr(h_stats), None, None, None, None, None,
                            None, None, _lib.ptr(h_best), _lib.ptr(h_abest), _lib.ptr(h_bpool))
    hstruct = hb.struct()

    def step_e2e():
        _lib.check(L.stw_plan_batch(C.byref(hstruct), C.byref(opts), C.byref(host_out), err, 1024), err)

    # warm-up + correctness of the run itself
    for _ in range(max(args.warmup, 1)):
        step_device()
    torch.cuda.synchronize(dev)
    rc = o_rc.cpu().numpy()
    stats = o_stats.cpu().numpy().reshape(T * Cn, _lib.NSTATS)
    if rc.max() != 0:
        raise SystemExit(f"planner reported errors on {int((rc != 0).sum())} units")
    planned = int(stats[:, 0].sum())  # static events given an address, summed over candidates
    events = N
    w = {"events": events, "unit_events": planned, "sort_records": events}

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # 256 MiB > 126 MB L2
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    def timed(fn, k, profile):
        total = 0.0
        if profile:
            _lib.profile_collect(reset=True)
            _lib.profile(True)
        launches0 = _lib.launch_count()
        for _ in range(k):
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            ev0.record(stream)
            fn()
            ev1.record(stream)
            torch.cuda.synchronize(dev)
            total += ev0.elapsed_time(ev1)
        launches = _lib.launch_count() - launches0
        prof = {}
        if profile:
            _lib.profile(False)
            prof = _lib.profile_collect(reset=True)
        return total / 1e3, launches, prof

    with ClockSampler(local) as clk:
        t_dev, launches, prof = timed(step_device, args.steps, True)
    t_plain, _, _ = timed(step_device, args.steps, False)  # unprofiled timing is the headline
    t_e2e, _, _ = timed(step_e2e, args.steps, False)

    def max_all(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_all(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    t_plain_max = max_all(t_plain)
    t_e2e_max = max_all(t_e2e)
    total_planned = sum_all(planned) * args.steps
    value = total_planned / t_plain_max
    e2e_value = total_planned / t_e2e_max

    # roofline of the dominant kernel (profiled run, same stream)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    top = max(prof.items(), key=lambda kv: kv[1][1]) if prof else ("?", (1, 0.0))
    kname, (kcount, kms) = top
    lps = kcount / max(args.steps, 1)
    avg_ms = kms / max(kcount, 1)
    abytes = algo_bytes(kname, w, lps)
    achieved = abytes / (avg_ms / 1e3) / 1e9 if avg_ms > 0 else float("nan")
    prof_total = sum(v[1] for v in prof.values())
    roofline = {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None, "avg_launch_ms": avg_ms,
                "share_of_kernel_time": kms / prof_total if prof_total else None,
                "peak_source": "measured" if "hbm_gbs" in peaks else "fallback"}
    if args.profile_print and rank == 0:
        for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
            print(f"{k:28s} launches {c:6d}  total {ms:9.3f} ms  avg {ms / c:8.4f} ms", file=sys.stderr)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = traces[:1024]
        dt, n_cpu = cpu_sweep(sample, threads)
        cpu = {"value": n_cpu / dt, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"oracle C port of the reference planner, first {len(sample)} c4 traces x 4 candidates"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_plain_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic: reference-exact c4 traces regenerated from seeds (rank r: seeds r*4096..)",
            "config": {"workload": "c4_batched_sweep", "traces_per_rank": T, "candidates": Cn,
                       "events_per_rank": N, "planned_allocs_per_step_per_rank": planned,
                       "parallelism": f"dp{world} (independent traces per rank)",
                       "l2": "256 MiB buffer written between timed steps (flush)", "trace_gen_s": round(t_gen, 2)},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": hb.nbytes,
                    "d2h_bytes_per_step": int(N * 8 + T * (4 + 8) + T * Cn * (4 + 16 + 8 * _lib.NSTATS))},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
