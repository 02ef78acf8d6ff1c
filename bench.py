#!/usr/bin/env python
"""Benchmark of the hot path: the batched planner sweep.

One step = plan 4096 reference-exact synthetic dense-model traces under the 4
(fusion, gap_insert) candidates, self-check every plan (static peak + the
rectangle sweep), pick the best candidate per trace -- i.e. 16,384 calls of
the reference's synthesize_static_plan -- and exchange the per-trace best
plans across the ranks (NCCL allreduce MIN over int64[4096] packed
(pool << 2 | cand), SUM of failing units).

Scaling: weak by default -- every rank plans its own c4-sized batch of 4096
traces (rank r: seeds r*4096..; rank 0's is exactly c4), so per-GPU work is
fixed and the job's sweep grows with N. `--scaling strong` splits c4's 4096
traces into contiguous blocks over the N ranks instead (its per-rank call is
latency-bound below ~2k traces).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl stw|reference]

`--gpus N` outside torchrun re-launches itself under torch.distributed.run
with N ranks (one process per GPU).

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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="stw", choices=["stw", "reference"])
    ap.add_argument("--traces", type=int, default=4096,
                    help="traces in the sweep (strong: split over the ranks; weak: per rank); c4 = 4096")
    ap.add_argument("--scaling", default="weak", choices=["strong", "weak"],
                    help="weak (default): every rank plans its own c4-sized batch (rank r: seeds r*4096..), "
                         "the whole job grows with N; strong: c4's 4096 traces split over the N GPUs")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend (gloo + --share-gpu: several ranks on one GPU, for tests)")
    ap.add_argument("--share-gpu", action="store_true", help="every rank uses cuda:0 (tests on a 1-GPU box)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernel-sweep", action="store_true", help="skip the K1/K7/K2 >>L2 roofline sweep")
    ap.add_argument("--sweep-reps", type=int, default=64, help="c4 copies in the K1/K7 sweep")
    ap.add_argument("--no-configs", action="store_true", help="skip the single-trace c1/c2/c3/c3b/c5 section")
    ap.add_argument("--profile-print", action="store_true", help="per-kernel table on stderr")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def seeds_of(rank: int, world: int, n: int, scaling: str) -> range:
    """The c4 seeds a rank plans: strong = a contiguous block of the n-trace
    sweep; weak = its own n traces."""
    if scaling == "weak":
        return range(rank * n, (rank + 1) * n)
    return range(rank * n // world, (rank + 1) * n // world)


def make_traces(seeds):
    from paper_2507_16274_b200 import tracegen

    return [tracegen.synth_arrays(tracegen.c4_config(s)) for s in seeds]


def self_launch(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-run under torch.distributed.run
    with N ranks (one process per GPU); rank 0 prints the line."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


# ---------------------------------------------------------------------------
# CPU side (oracle port of the reference planner)

_POOL_TRACES = {}  # seed -> TraceArrays, filled before the pool forks (workers inherit it)


def _pool_plan(seeds):
    """One pool task: plan the seeds' traces under the 4 candidates with the C oracle."""
    from oracle import oracle as O

    n = 0
    for s in seeds:
        ta = _POOL_TRACES[s]
        for f, g in CANDS:
            r = O.plan(ta, f, g)
            assert r.rc == 0, r.err
            n += r.stats["num_events"]
    return n


class CpuSweep:
    """The reference planner's CPU cost on this host: the C port of the
    reference (oracle/) over c4 traces x 4 candidates, one process per host
    core (multiprocessing.Pool); the traces are generated
    before the pool forks, so no timed call pays for them."""

    def __init__(self, seeds, procs=None, traces=None):
        import multiprocessing as mp

        from oracle import oracle as O

        self.procs = procs or os.cpu_count() or 1
        seeds = list(seeds)
        for s, ta in zip(seeds, traces if traces is not None else make_traces(seeds)):
            _POOL_TRACES[s] = ta
        O.lib()  # loaded once, inherited by the workers
        k = self.procs * 4  # tasks: contiguous chunks, four per worker
        self.chunks = [seeds[i * len(seeds) // k:(i + 1) * len(seeds) // k] for i in range(k)]
        self.pool = mp.get_context("fork").Pool(self.procs)
        self.pool.map(_pool_plan, [c[:1] for c in self.chunks if c])  # every worker started and warm

    def run(self):
        """(seconds, planned allocations) of one full pass."""
        t0 = time.perf_counter()
        total = sum(self.pool.map(_pool_plan, self.chunks))
        return time.perf_counter() - t0, total

    def close(self):
        self.pool.terminate()
        self.pool.join()


def host_info() -> dict:
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    import platform

    return {"cpu_model": model, "cpu_count": os.cpu_count(), "python": platform.python_version()}


def run_reference(args, rank, world):
    """The reference arm: the C port of the reference planner (oracle/) on every
    host core, on this run's config (the c4 sweep). Under torchrun only rank 0
    works; the others exit."""
    if rank != 0:
        return
    cpu = CpuSweep(range(args.traces))
    try:
        for _ in range(max(args.warmup - 1, 0)):
            cpu.run()
        times, total = [], 0
        for _ in range(args.steps):
            dt, total = cpu.run()
            times.append(dt)
    finally:
        cpu.close()
    t = sum(times)
    value = total * args.steps / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int64",
        "data": "synthetic: reference-exact c4 traces (seeds 0..4095) regenerated from seeds",
        "config": {"workload": "c4_batched_sweep", "traces": args.traces, "candidates": 4,
                   "planned_allocs_per_step": total},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu.procs, "kind": "port",
                         "sample": f"full c4 sweep ({args.traces} traces x 4 candidates) per step, "
                                   f"multiprocessing.Pool({cpu.procs})", **host_info()},
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
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # the sampler is live before the timed region starts
            while not self.lines and time.time() - t0 < 5 and self.proc.poll() is None:
                time.sleep(0.005)
            self.first = len(self.lines)  # samples from here on fall inside the region
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            t0 = time.time()  # one sample at (or just after) the end of the region
            n = len(self.lines)
            while len(self.lines) == n and time.time() - t0 < 1 and self.proc.poll() is None:
                time.sleep(0.002)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines[getattr(self, "first", 0):]:
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


_SM_MAX = []


def sm_max_mhz():
    """The GPU's maximum SM clock (nvidia-smi, queried once; B200: 1965 MHz)."""
    if not _SM_MAX:
        v = None
        try:
            r = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits"],
                               capture_output=True, text=True, timeout=20)
            v = float(r.stdout.strip().splitlines()[0])
        except (OSError, ValueError, IndexError, subprocess.SubprocessError):
            v = 1965.0
        _SM_MAX.append(v)
    return _SM_MAX[0]


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# algorithmic bytes per launch; w = workload counts of one step
def algo_bytes(kernel: str, w: dict, launches_per_step: float) -> float:
    per_step = {
        # planner layers (K5/K6): 32 B/item in + 8 B/item out, per unit
        "k_layers": 40.0 * w["unit_items"],
        "k_layers_w32": 40.0 * w["unit_items"],
        # K7 fast path: 24 B per rectangle of each candidate plan
        "k_overlap_sweep": 24.0 * w["unit_events"],
        "k_validate_tiles": 24.0 * w["unit_events"],
        # fusion: the trace's events are read once per attempt at least
        "k_fusion": 32.0 * w["events"],
        # K1: 17 B/event (t_s, t_e, size, dyn)
        "k_peak_warp": 17.0 * w["events"],
        # segmented sorts: 12 B/record read + written per sort
        "k_seg_radix<8>": 24.0 * w["events"],
        "k_emit": 40.0 * w["unit_events"],
    }.get(kernel)
    if per_step is None:
        return float("nan")
    return per_step / max(launches_per_step, 1.0)


# ---------------------------------------------------------------------------
# HBM roofline sweep of the data-parallel kernels (inputs >> L2)

def kernel_sweep(dev, db, hb, planned_addr, reps: int, hbm: float):
    """K1 (peak live bytes), K7 (validate_plan over many plans) and K2 (radix
    sort) on inputs far larger than the 126 MB L2, each timed on its stream
    with CUDA events (K1/K7: the library's per-launch events around the
    kernel; K2: the whole multi-pass call). Returns {kernel: stats}."""
    import torch

    from paper_2507_16274_b200 import _lib, api

    L = _lib.load()
    err = _lib.errbuf()
    stream = torch.cuda.current_stream(dev)
    sh = C.c_void_p(stream.cuda_stream)
    out = {}

    def kernel_ms(fn, name, iters=3):
        fn()
        torch.cuda.synchronize(dev)
        _lib.profile_collect(reset=True)
        _lib.profile(True)
        torch.cuda.nvtx.range_push("sweep_" + name.split("<")[0])  # ncu --nvtx --nvtx-include sweep_<kernel>/ selects these
        for _ in range(iters):
            fn()
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize(dev)
        _lib.profile(False)
        prof = _lib.profile_collect(reset=True)
        cnt, ms = prof[name]
        return ms / cnt

    def entry(name, records, unit_bytes, ms, note, traffic_key=None, launches=1):
        gbs = records * unit_bytes / (ms / 1e3) / 1e9
        tr = ncu_traffic(traffic_key) if traffic_key else None
        out[name] = {"kernel": name, "records": int(records), "algorithmic_bytes_per_record": unit_bytes,
                     "ms": ms, "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                     "traffic": tr["bytes"] * launches if tr else None,
                     "traffic_source": tr["source"] if tr else None, "what": note}
        if tr and tr.get("inst"):
            out[name]["issue"] = issue_roofline(tr["inst"], ms / launches, sm_max_mhz())

    # K1: R copies of the c4 batch (static_only, as the planner's self-check)
    T, N = db.T, db.N
    t = db.t
    cols = {k: t[k].repeat(reps) for k in ("size", "t_s", "t_e", "dyn")}
    ev_off = torch.cat([db.ev_off[:-1] + r * N for r in range(reps)] + [db.ev_off[-1:] + (reps - 1) * N])
    horizon, n_sched = db.horizon.repeat(reps), db.n_sched.repeat(reps)
    bk1 = _lib.Batch(T * reps, 1, N * reps, _lib.ptr(ev_off), _lib.ptr(t["id"]), _lib.ptr(cols["size"]),
                     _lib.ptr(cols["t_s"]), _lib.ptr(cols["t_e"]), _lib.ptr(t["ps"]), _lib.ptr(t["pe"]),
                     _lib.ptr(cols["dyn"]), _lib.ptr(horizon), _lib.ptr(n_sched))
    peaks = np.zeros(T * reps, np.int64)

    def k1():
        _lib.check(L.stw_peak_live(C.byref(bk1), 1, _lib.ptr(peaks), sh, err, 1024), err)

    ms = kernel_ms(k1, "k_peak_warp")
    entry("k_peak_warp", N * reps, 17.0, ms, f"K1 peak live bytes, {reps}x c4 ({N * reps} events); "
          "17 B/event read (t_s, t_e, size, dyn), timeline in shared memory", "k_peak_warp@sweep")
    del cols, ev_off, horizon, n_sched

    # K7: the c4 plans of all 4 candidates, sweep-ordered, R copies
    stat = np.concatenate([tr.dyn == 0 for tr in hb.traces])
    keep = torch.from_numpy(np.flatnonzero(stat)).to(dev)
    cnt = torch.from_numpy(np.asarray([int((tr.dyn == 0).sum()) for tr in hb.traces], np.int64))
    off1 = torch.zeros(T + 1, dtype=torch.int64)
    off1[1:] = torch.cumsum(cnt, 0)
    n1 = int(off1[-1])
    off = torch.cat([off1[:-1] + r * n1 for r in range(reps)] + [off1[-1:] + (reps - 1) * n1]).to(dev)
    ts, te, sz = (t[k].index_select(0, keep).repeat(reps) for k in ("t_s", "t_e", "size"))
    ad = planned_addr.index_select(1, keep).repeat(1, reps).contiguous()
    nc = ad.shape[0]
    count = [None]

    def k7():
        count[0] = api.validate_sets(off, ts, te, sz, ad, 9)

    ms = kernel_ms(k7, "k_overlap_sweep")
    assert int(count[0].abs().sum()) == 0, "planner output failed validation"
    entry("k_overlap_sweep", n1 * reps * nc, 24.0, ms,
          f"K7 validate_plan of {T * reps * nc} plans ({n1 * reps} rectangles x {nc} candidates); "
          "SURVEY §8(d4): 24 B per rectangle of each plan (addr, size, t_s, t_e); the kernel reads the shared "
          "size/t_s/t_e once per set, so DRAM traffic is ~12 B per (rectangle, candidate)",
          "k_overlap_sweep@sweep")
    del ts, te, sz, ad, off

    # K2: 2^27 (u64 key, u32 value) pairs, 42-bit keys (c5's widest sort: 6 passes)
    n2 = 1 << 27
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    keys0 = torch.randint(0, 1 << 42, (n2,), dtype=torch.int64, device=dev, generator=g)
    keys = torch.empty_like(keys0)
    vals = torch.empty(n2, dtype=torch.int32, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for it in range(4):
        keys.copy_(keys0)
        torch.arange(n2, dtype=torch.int32, device=dev, out=vals)
        torch.cuda.synchronize(dev)
        if it:
            torch.cuda.nvtx.range_push("sweep_radix_sort_pairs")
        e0.record(stream)
        api.radix_sort_pairs(keys, vals, 0, 42, stream)
        e1.record(stream)
        if it:
            torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize(dev)
        if it:
            tot += e0.elapsed_time(e1)
    ms = tot / 3
    assert bool((keys[1:] >= keys[:-1]).all()), "radix sort output not sorted"
    passes = 6
    entry("radix_sort_pairs", n2, 24.0 * passes, ms,
          f"K2 stable LSD radix sort of {n2} (u64, u32) pairs on 42 key bits ({passes} passes); "
          "24 B/record/pass (key + value read and written); traffic = 6 passes (+ the 8 B/record histogram read)",
          "k_os_pass@sweep", passes)
    del keys0, keys, vals

    # the look-back scan (every prefix sum of the path): 2^28 int64 in place; 16 B/element
    n3 = 1 << 28
    xs = torch.randint(0, 1 << 20, (n3,), dtype=torch.int64, device=dev, generator=g)
    want = torch.cumsum(xs[: 1 << 20], 0)
    ys = torch.empty_like(xs)

    def scan():
        api.scan_i64(xs, ys, True, stream)

    ms = kernel_ms(scan, "k_scan_lb<T>")
    assert torch.equal(ys[: 1 << 20], want), "scan output"
    entry("k_scan_lb", n3, 16.0, ms, f"device-wide inclusive prefix sum of {n3} int64 (decoupled look-back, "
          "single pass): 8 B read + 8 B written per element", "k_scan_lb@sweep")
    del xs, ys, want
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# single-trace configs: plan / replay / baseline on the device,
# replay ops/s and the bit-exact fragmentation ratios

STAGES = ("plan", "reuse", "validate", "simulate", "baseline", "peak")


def config_sweep(names, reps: int = 3, cpu: bool = True):
    """Per config, per stage (synthesize_static_plan,
    derive_reuse_map, validate_plan, simulate, run_baseline, peak_live_bytes):
    the device path through the package API (host arrays in, host objects /
    columns out), best of `reps`, beside the C port of the reference (oracle/,
    one host thread) on the same inputs in the same run -- plus the
    bit-exact fragmentation ratios."""
    import paper_2507_16274_b200 as M
    from paper_2507_16274_b200 import api, tracegen

    if cpu:
        from oracle import oracle as O

    def best(fn, k=reps):
        t, r = float("inf"), None
        for _ in range(k):
            t0 = time.perf_counter()
            r = fn()
            t = min(t, time.perf_counter() - t0)
        return t, r

    out = {}
    for name in names:
        ta = tracegen.synth_arrays(tracegen.config(name))
        tr = M.Trace.from_arrays(ta)
        g = {}
        g["plan"], plan = best(lambda: M.synthesize_static_plan(tr))
        g["reuse"], rmap = best(lambda: M.derive_reuse_map(plan, tr))
        c = plan.columns()
        g["validate"], _pairs = best(lambda: api.validate_columns(c.id, c.addr, c.size, c.t_s, c.t_e))
        bundle = plan.to_bundle(rmap)
        g["simulate"], (rep, _log) = best(lambda: M.simulate(tr, bundle))
        g["baseline"], base = best(lambda: M.run_baseline(tr))
        g["peak"], peak = best(lambda: M.peak_live_bytes(ta))
        # the same plan from a trace of event objects, as the reference's
        # parse_trace / synth_trace hand it over: the tensorising walk is timed too
        from paper_2507_16274_b200.domain import Trace as _ObjTrace

        objs = _ObjTrace(tuple(tr.events), tr.phase_schedule, tr.layer_schedule)
        t_obj, plan_obj = best(lambda: M.synthesize_static_plan(objs), 1)
        assert plan_obj.pool_size == plan.pool_size
        del objs, plan_obj
        n = len(ta)
        row = {"events": n, "pool_size": int(plan.pool_size),
               "planned_allocs_per_s": int((ta.dyn == 0).sum()) / g["plan"],
               "replay_ops_per_s": 2 * n / g["simulate"],
               "fragmentation": rep.fragmentation, "efficiency": rep.efficiency,
               "baseline_fragmentation": base.fragmentation,
               "fallbacks": int(rep.fallback_count), "reuse_hits": int(rep.reuse_hits),
               "gpu_ms": {k: 1e3 * v for k, v in g.items()},
               "plan_from_event_objects_ms": 1e3 * t_obj}
        if cpu:
            keys, kidx = ta.dynamic_keys()
            t_lo = np.asarray([rmap.entries[k].t_lo for k in keys], np.int64)
            t_hi = np.asarray([rmap.entries[k].t_hi for k in keys], np.int64)
            h = {}
            h["plan"], op = best(lambda: O.plan(ta), 1)
            h["reuse"], (off, lo, hi) = best(lambda: O.reuse(c.addr, c.size, c.t_s, c.t_e, t_lo, t_hi), 1)
            h["validate"], _ = best(lambda: O.validate(c.id, c.addr, c.size, c.t_s, c.t_e), 1)
            key = np.where(kidx >= 0, kidx, -1).astype(np.int32)
            h["simulate"], orep = best(lambda: O.simulate(ta, key, plan.pool_size, 512, c.id, c.addr, c.size, c.t_s,
                                                          c.t_e, off, lo, hi, True), 1)
            h["baseline"], obase = best(lambda: O.baseline(ta), 1)
            h["peak"], opeak = best(lambda: O.peak_live(ta.size, ta.t_s, ta.t_e), 1)
            assert op.stats["pool_size"] == plan.pool_size and opeak == peak
            assert orep.report == rep.to_dict() and obase.report == base.to_dict(), name
            row["cpu_ms"] = {k: 1e3 * v for k, v in h.items()}
            row["cpu_over_gpu"] = {k: h[k] / g[k] for k in STAGES}
        out[name] = row
    return out


def ncu_traffic(key):
    """DRAM bytes per launch of `key` from the committed `ncu --set full` capture
    (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            e = json.load(fh).get(key)
    except (OSError, ValueError):
        return None
    return None if e is None else {"bytes": e["dram_bytes_per_launch"], "source": e["capture"],
                                   "inst": e.get("warp_inst_per_launch")}


def issue_roofline(inst_per_launch, ms, sm_mhz):
    """Instruction-issue roofline of a kernel that is not byte-bound: warp
    instructions per launch (ncu smsp__inst_executed of the committed capture)
    over the CUDA-event launch time, against one warp instruction per cycle per
    scheduler (148 SMs x 4 schedulers) at the measured SM clock."""
    if not inst_per_launch or not ms or not sm_mhz:
        return None
    achieved = inst_per_launch / (ms / 1e3)
    peak = 148 * 4 * sm_mhz * 1e6
    return {"achieved": achieved, "peak": peak, "unit": "warp-inst/s", "frac": achieved / peak,
            "warp_inst_per_launch": inst_per_launch}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args))
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)  # rank 0 alone runs the CPU reference; no collective
        return

    import torch

    from paper_2507_16274_b200 import _lib, api
    from paper_2507_16274_b200.batching import HostBatch

    if args.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    L = _lib.load()

    t_gen = time.perf_counter()
    seeds = seeds_of(rank, world, args.traces, args.scaling)
    traces = make_traces(seeds)
    t_gen = time.perf_counter() - t_gen
    n_sweep = args.traces if args.scaling == "strong" else args.traces * world  # traces of the whole job
    hb = HostBatch(traces, pinned=True)
    db = hb.to_device(dev)
    # the pinned host batch also keeps its compact columns (id as int32 offsets,
    # size in power-of-two units; made once, outside the timed region):
    # stw_plan_batches uploads those (25 instead of 33 B/event) and widens on the device
    packed = hb.pack()
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
    o_addr = torch.empty((Cn, N), dtype=torch.int64, device=dev)  # every candidate's plan (validated in the sweep)
    dev_out = _lib.PlanOut(1, _lib.ptr(o_rc), _lib.ptr(o_err), _lib.ptr(o_stats), _lib.ptr(o_addr), None, None,
                           None, None, None, None, _lib.ptr(o_best), _lib.ptr(o_abest), _lib.ptr(o_bpool))
    opts = _lib.PlanOpts(Cn, 1, _lib.ptr(cb), 512, sh)
    dstruct = db.struct()
    err = _lib.errbuf()

    # the sweep's one exchange: the best plan of every trace of the
    # job as packed (pool << 2 | cand), INT64_MAX outside this rank's block,
    # allreduce MIN over int64[n_sweep] (ties -> lowest candidate, the
    # reference's order); the failing units' count, allreduce SUM
    g_keys = torch.empty(n_sweep, dtype=torch.int64, device=dev)
    g_bad = torch.zeros(1, dtype=torch.int64, device=dev)
    off0 = seeds.start
    i64max = torch.iinfo(torch.int64).max

    def allreduce(t, op):
        if world == 1:
            return
        if args.backend == "gloo":
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op)

    def combine(bpool, best, rc):
        g_keys.fill_(i64max)
        g_keys[off0:off0 + T].copy_((bpool.to(dev, non_blocking=True) << 2) | best.to(dev, torch.int64,
                                                                                    non_blocking=True))
        g_bad.copy_((rc.to(dev, non_blocking=True) != 0).sum().view(1))
        if world > 1:
            allreduce(g_keys, dist.ReduceOp.MIN)
            allreduce(g_bad, dist.ReduceOp.SUM)

    def step_device():
        _lib.check(L.stw_plan_batch(C.byref(dstruct), C.byref(opts), C.byref(dev_out), err, 1024), err)
        combine(o_bpool, o_best, o_rc)

    # host-side buffers for the end-to-end path (pinned in, pinned out)
    h_rc = torch.empty(T * Cn, dtype=torch.int32).pin_memory()
    h_err = torch.empty(2 * T * Cn, dtype=torch.int64).pin_memory()
    h_stats = torch.empty(T * Cn * _lib.NSTATS, dtype=torch.int64).pin_memory()
    h_best = torch.empty(T, dtype=torch.int32).pin_memory()
    h_bpool = torch.empty(T, dtype=torch.int64).pin_memory()
    h_abest = torch.empty(N, dtype=torch.int64).pin_memory()
    host_out = _lib.PlanOut(0, _lib.ptr(h_rc), _lib.ptr(h_err), _lib.ptr(h_stats), None, None, None, None, None,
                            None, None, _lib.ptr(h_best), _lib.ptr(h_abest), _lib.ptr(h_bpool))
    # one host output set per lane: stw_plan_batches plans step k in lane
    # k % lanes, concurrently with the other lanes, so steps of different lanes
    # must not share result buffers
    lanes = int(os.environ.get("STW_LANES", "2"))
    hsets = [(h_rc, h_err, h_stats, h_best, h_abest, h_bpool)]
    for _ in range(1, max(lanes, 1)):
        hsets.append(tuple(torch.empty_like(x).pin_memory() for x in hsets[0]))
    houts = [_lib.PlanOut(0, _lib.ptr(a), _lib.ptr(b_), _lib.ptr(c), None, None, None, None, None, None, None,
                          _lib.ptr(d), _lib.ptr(e), _lib.ptr(f)) for a, b_, c, d, e, f in hsets]
    hstruct = hb.struct()

    def step_e2e():
        _lib.check(L.stw_plan_batch(C.byref(hstruct), C.byref(opts), C.byref(host_out), err, 1024), err)
        combine(h_bpool, h_best, h_rc)

    def e2e_pipelined(k):
        """K steps through stw_plan_batches: every step copies its batch from pinned
        host memory and its results back, double-buffered so step i+1's upload
        and step i-1's download overlap step i's planning. Device time (events
        on the launching stream around the whole call, which joins its copy
        stream before returning); the L2 is flushed before the call."""
        bs = (_lib.Batch * k)(*([hstruct] * k))
        os_ = (_lib.PlanOut * k)(*[houts[i % len(houts)] for i in range(k)])
        flush.zero_()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        ev0.record(stream)
        _lib.check(L.stw_plan_batches(k, bs, C.byref(opts), os_, err, 1024), err)
        for i in range(k):  # every step's results go through the exchange
            hs = hsets[i % len(hsets)]
            combine(hs[5], hs[3], hs[0])
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        return ev0.elapsed_time(ev1) / 1e3

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
    items = int(stats[:, 3].sum() + stats[:, 4].sum() - stats[:, 6].sum())  # plans + residuals - fused away
    w = {"events": events, "unit_events": planned, "unit_items": items}

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
            torch.cuda.nvtx.range_push("bench_step")  # ncu --nvtx --nvtx-include bench_step/ selects the step
            ev0.record(stream)
            fn()
            ev1.record(stream)
            torch.cuda.nvtx.range_pop()
            torch.cuda.synchronize(dev)
            total += ev0.elapsed_time(ev1)
        launches = _lib.launch_count() - launches0
        prof = {}
        if profile:
            _lib.profile(False)
            prof = _lib.profile_collect(reset=True)
        return total / 1e3, launches, prof

    step_e2e()  # warm-up of the host-buffer path (its input staging grows the memory pool once)
    e2e_pipelined(2)  # warm-up of the pipelined path
    with ClockSampler(local) as clk:  # clocks sampled (every 20 ms) across all the timed regions
        t_dev, launches, prof = timed(step_device, args.steps, True)
        t_plain, _, _ = timed(step_device, args.steps, False)  # unprofiled timing is the headline
        t_e2e_serial, _, _ = timed(step_e2e, args.steps, False)
        t_e2e = e2e_pipelined(args.steps)

    def reduce_scalar(x, op):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        allreduce(t, op)
        return float(t.item())

    t_plain_max = reduce_scalar(t_plain, dist.ReduceOp.MAX if world > 1 else None)
    t_e2e_max = reduce_scalar(t_e2e, dist.ReduceOp.MAX if world > 1 else None)
    t_e2e_serial_max = reduce_scalar(t_e2e_serial, dist.ReduceOp.MAX if world > 1 else None)
    total_planned = reduce_scalar(planned, dist.ReduceOp.SUM if world > 1 else None) * args.steps
    value = total_planned / t_plain_max
    e2e_value = total_planned / t_e2e_max

    # the exchange's result, checked against the reference's c4 anchor (sum of
    # the best pools over seeds 0..4095, tests/golden/anchors.json)
    step_device()
    torch.cuda.synchronize(dev)
    keys = g_keys.cpu().numpy()
    verified = None
    if n_sweep >= 4096:
        with open(os.path.join(ROOT, "tests", "golden", "anchors.json")) as fh:
            want = json.load(fh)["c4"]["sum_best_pool"]
        got = int((keys[:4096] >> 2).sum())
        verified = {"c4_sum_best_pool": got, "matches_reference": got == want,
                    "failing_units": int(g_bad.item())}
        if got != want or int(g_bad.item()):
            raise SystemExit(f"sweep result differs from the reference anchor: {verified}")

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
    tr = ncu_traffic(kname)
    roofline = {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": tr["bytes"] if tr else None,
                "algorithmic_bytes_per_launch": abytes, "traffic_source": tr["source"] if tr else None,
                "avg_launch_ms": avg_ms,
                "share_of_kernel_time": kms / prof_total if prof_total else None,
                "peak_source": "measured" if "hbm_gbs" in peaks else "fallback",
                "issue": issue_roofline(tr.get("inst") if tr else None, avg_ms, sm_max_mhz())}
    if args.profile_print and rank == 0:
        for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
            print(f"{k:28s} launches {c:6d}  total {ms:9.3f} ms  avg {ms / c:8.4f} ms", file=sys.stderr)

    sweep = None
    if not args.no_kernel_sweep and world == 1:
        sweep = kernel_sweep(dev, db, hb, o_addr, args.sweep_reps, hbm)
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = config_sweep(["c1_llama2_7b_1f1b", "c2_llama2_7b_vpp_rcp", "c3_mixtral_moe", "c3b_mixtral_moe_rcp",
                                "c5_llama3_70b"], cpu=not args.no_cpu_baseline)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        k = min(1024, len(traces))
        sweep_cpu = CpuSweep(seeds[:k], traces=traces[:k])
        try:
            dt, n_cpu = sweep_cpu.run()
        finally:
            sweep_cpu.close()
        cpu = {"value": n_cpu / dt, "unit": UNIT, "cores": sweep_cpu.procs, "kind": "port",
               "sample": f"oracle C port of the reference planner, c4 seeds 0..{k - 1} x 4 candidates, "
                         f"multiprocessing.Pool({sweep_cpu.procs})", **host_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_plain_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int64",
            "data": "synthetic: reference-exact c4 traces regenerated from their seeds",
            "config": {"workload": "c4_batched_sweep", "traces": n_sweep, "traces_per_rank": T, "candidates": Cn,
                       "events_per_rank": N, "planned_allocs_per_step_per_rank": planned,
                       "parallelism": f"dp{world}: " + ("the sweep's traces in contiguous blocks per rank"
                                                         if args.scaling == "strong" else "own traces per rank")
                       + "; allreduce MIN over int64[traces] of (pool << 2 | cand) + SUM of failing units per step",
                       "backend": args.backend if world > 1 else None,
                       "l2": "256 MiB buffer written between timed steps (flush)", "trace_gen_s": round(t_gen, 2)},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": hb.upload_nbytes, "compact_upload": packed,
                    "d2h_bytes_per_step": int(N * 8 + T * (4 + 8) + T * Cn * (4 + 16 + 8 * _lib.NSTATS)),
                    "how": "stw_plan_batches over the K steps: pinned host batch in, host results out every step, "
                           "double-buffered staging (copies overlap the neighbouring steps' planning); even and odd steps "
                           "in two concurrent lanes (threads/streams) that fill each other's host round trips",
                    "serial_value": total_planned / t_e2e_serial_max,
                    "serial_how": "one synchronous stw_plan_batch call per step with host buffers"},
            "gpu_launches": int(launches),
            "verified": verified,
            "roofline": roofline,
            "kernel_roofline": sweep,
            "configs": configs,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
