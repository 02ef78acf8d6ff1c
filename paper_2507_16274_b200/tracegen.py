"""Synthetic training traces emitted straight into the SoA layout.

This is the input side of the hot path: it reproduces the
reference generator's traces event for event (`memplan/synth.py:263-366`,
same `random.Random` draw sequence per seed) so that the pinned configs can
be rebuilt on the GPU box, where `/root/reference` does not exist, and fed to
the device without ever creating per-event Python objects.

The recorder model: every alloc/free is one record, so the record index is
the timestamp; alloc ids are handed out in record order, which makes the
(t_s, id) event order equal to id order (`synth.py:116-203`).
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from .domain import DEFAULT_ALIGNMENT, MemplanError, PhaseId, PhaseKind, Trace, align_up
from .soa import TraceArrays

MIB = 1 << 20
DEFAULT_PALETTE = tuple(n * MIB for n in (2, 3, 4, 6, 8, 12, 16, 24))
PRESETS = ("dense", "dense_recompute", "dense_vpp", "dense_vpp_recompute", "moe", "moe_recompute")
MOE_LAYER_STRIDE = 2  # synth.py:45
MOE_TENSORS_PER_LAYER = 2  # synth.py:46


class SynthConfigError(MemplanError):
    pass


@dataclass(frozen=True)
class SynthConfig:
    """Generator knobs (synth.py:53-113)."""

    preset: str
    num_layers: int = 12
    num_microbatches: int = 4
    num_chunks: int = 1
    size_palette: tuple = DEFAULT_PALETTE
    distinct_sizes: int = len(DEFAULT_PALETTE)
    persistent_bytes: int = 1024 * MIB
    transient_ratio: float = 0.3
    moe_size_range: tuple = (1 * MIB, 12 * MIB)
    seed: int = 0
    alignment: int = DEFAULT_ALIGNMENT

    @property
    def recompute(self) -> bool:
        return self.preset.endswith("_recompute")

    @property
    def vpp(self) -> bool:
        return "vpp" in self.preset

    @property
    def moe(self) -> bool:
        return self.preset.startswith("moe")

    @classmethod
    def for_preset(cls, preset: str, **overrides) -> "SynthConfig":
        if preset not in PRESETS:
            raise SynthConfigError(f"unknown preset {preset!r}")
        if "vpp" in preset:
            overrides.setdefault("num_chunks", 2)
        cfg = cls(preset=preset, **overrides)
        cfg.validate()
        return cfg

    def validate(self) -> None:
        checks = [
            (self.preset in PRESETS, f"unknown preset {self.preset!r}"),
            (self.distinct_sizes == len(self.size_palette), "distinct_sizes must equal len(size_palette)"),
            (all(s > 0 and s % self.alignment == 0 for s in self.size_palette),
             "palette sizes must be positive and aligned"),
            (self.num_chunks >= 1, "num_chunks must be >= 1"),
            (not self.vpp or self.num_chunks >= 2, "vpp presets need num_chunks >= 2"),
            (self.vpp or self.num_chunks == 1, "non-vpp presets use num_chunks = 1"),
            (self.num_layers >= self.num_chunks, "need at least one layer per chunk"),
            (self.num_microbatches >= 1, "num_microbatches must be >= 1"),
            (self.persistent_bytes >= (self.num_layers + 2) * self.alignment,
             "persistent_bytes too small to split"),
            (self.transient_ratio >= 0, "transient_ratio must be >= 0"),
        ]
        for ok, msg in checks:
            if not ok:
                raise SynthConfigError(msg)
        if self.moe:
            lo, hi = self.moe_size_range
            if not (0 < lo <= hi):
                raise SynthConfigError("moe_size_range must satisfy 0 < min <= max")


def phase_order(cfg: SynthConfig) -> list:
    """(kind, microbatch, chunk) in execution order (synth.py:206-226)."""
    M, C = cfg.num_microbatches, cfg.num_chunks
    if not cfg.vpp:
        return [step for m in range(M) for step in (("F", m, 0), ("B", m, 0))]
    w = min(2, M)
    order = [("F", m, c) for c in range(C) for m in range(w)]
    fwd = [("F", m, c) for m in range(w, M) for c in range(C)]
    bwd = [("B", m, c) for m in range(M) for c in range(C - 1, -1, -1)]
    for k, f in enumerate(fwd):
        order += [bwd[k], f]
    return order + bwd[len(fwd):]


class _Tape:
    """Record-dense op tape writing event columns indexed by id."""

    def __init__(self, cap_hint: int = 1024) -> None:
        self.t = 0
        self.size: list = []
        self.t_s: list = []
        self.t_e: list = []
        self.ps: list = []
        self.pe: list = []
        self.ls: list = []
        self.le: list = []
        self.mod: list = []  # alloc module per id (dynamic only)
        self.phase = -1
        self.phases: list = []
        self.starts: list = []
        self.ends: list = []
        self.lay_lo: dict = {}
        self.lay_hi: dict = {}

    def begin(self, pid: PhaseId) -> None:
        self._close()
        self.phases.append(pid)
        self.starts.append(self.t)
        self.phase = len(self.phases) - 1

    def _close(self) -> None:
        if self.phase >= 0:
            if self.t == self.starts[self.phase]:
                raise SynthConfigError(f"phase {self.phases[self.phase]} emitted no records")
            self.ends.append(self.t)

    def _touch(self, name: str) -> None:
        self.lay_lo.setdefault(name, self.t)
        self.lay_hi[name] = self.t + 1

    def alloc(self, size: int, module: str = None) -> int:
        rid = len(self.size)
        self.size.append(size)
        self.t_s.append(self.t)
        self.t_e.append(-1)
        self.ps.append(self.phase)
        self.pe.append(-1)
        self.mod.append(module)
        self.ls.append(module)
        self.le.append(None)
        if module is not None:
            self._touch(module)
        self.t += 1
        return rid

    def free(self, rid: int, module: str = "") -> None:
        if self.mod[rid] is not None:
            end_mod = module or self.mod[rid]
            self.le[rid] = end_mod
            self._touch(end_mod)
        self.t_e[rid] = self.t
        self.pe[rid] = self.phase
        self.t += 1

    def finish(self) -> TraceArrays:
        self._close()
        horizon = self.t
        last = len(self.phases) - 1
        t_e = np.asarray(self.t_e, dtype=np.int64)
        pe = np.asarray(self.pe, dtype=np.int64)
        open_ = t_e < 0
        t_e[open_] = horizon
        pe[open_] = last
        names = sorted(self.lay_lo)
        lidx = {n: i for i, n in enumerate(names)}
        n = len(self.size)
        dyn = np.asarray([m is not None for m in self.mod], dtype=np.uint8)
        ls = np.asarray([-1 if m is None else lidx[m] for m in self.ls], dtype=np.int32)
        le = np.asarray([-1 if m is None else lidx[m] for m in self.le], dtype=np.int32)
        return TraceArrays(
            id=np.arange(n, dtype=np.int64),
            size=np.asarray(self.size, dtype=np.int64),
            t_s=np.asarray(self.t_s, dtype=np.int32),
            t_e=t_e.astype(np.int32),
            ps=np.asarray(self.ps, dtype=np.int32),
            pe=pe.astype(np.int32),
            dyn=dyn,
            ls=ls,
            le=le,
            phases=list(self.phases),
            phase_start=np.asarray(self.starts, dtype=np.int64),
            phase_end=np.asarray(self.ends, dtype=np.int64),
            layer_names=names,
            layer_start=np.asarray([self.lay_lo[k] for k in names], dtype=np.int64),
            layer_end=np.asarray([self.lay_hi[k] for k in names], dtype=np.int64),
            n_known_layers=len(names),
        )


def synth_arrays(cfg: SynthConfig) -> TraceArrays:
    """Generate the trace for `cfg` directly as SoA (synth.py:263-366 semantics)."""
    cfg.validate()
    rng = random.Random(cfg.seed)
    tape = _Tape()
    pal = cfg.size_palette
    L, C = cfg.num_layers, cfg.num_chunks
    rc = cfg.recompute
    whole = int(cfg.transient_ratio)
    frac = cfg.transient_ratio - whole

    def layer_size(l: int) -> int:
        return pal[l % len(pal)]

    def transients() -> None:
        n = whole + (1 if rng.random() < frac else 0)
        for _ in range(n):
            tape.free(tape.alloc(rng.choice(pal)))

    def moe_size() -> int:
        lo, hi = cfg.moe_size_range
        return align_up(rng.randint(lo, hi), cfg.alignment)

    def is_moe(l: int) -> bool:
        return cfg.moe and l % MOE_LAYER_STRIDE == 1

    # persistent blocks (synth.py:234-240)
    tape.begin(PhaseId(PhaseKind.INIT))
    nb = L + 2
    blk = align_up(max(cfg.persistent_bytes // nb, cfg.alignment), cfg.alignment)
    for _ in range(nb - 1):
        tape.alloc(blk)
    tape.alloc(align_up(max(cfg.persistent_bytes - blk * (nb - 1), cfg.alignment), cfg.alignment))

    held: dict = {}  # (m, c) -> activation ids, alloc order
    experts: dict = {}  # (layer, m) -> open dynamic ids
    shards: list = []
    last_mb = cfg.num_microbatches - 1

    for kind, m, c in phase_order(cfg):
        layers = range(c * L // C, (c + 1) * L // C)
        if kind == "F":
            tape.begin(PhaseId(PhaseKind.FORWARD, m, c))
            prev = None
            for l in layers:
                act = tape.alloc(layer_size(l))
                transients()
                if is_moe(l):
                    inst = f"L{l:02d}.moe.F{m}"
                    ids = [tape.alloc(moe_size(), inst) for _ in range(MOE_TENSORS_PER_LAYER)]
                    if rc:
                        for rid in ids:
                            tape.free(rid, inst)
                    else:
                        experts[(l, m)] = ids
                if rc:
                    if prev is not None:
                        tape.free(prev)
                    prev = act
                else:
                    held.setdefault((m, c), []).append(act)
            if rc and prev is not None:
                tape.free(prev)
        else:
            tape.begin(PhaseId(PhaseKind.BACKWARD, m, c))
            prev = None
            acts = None if rc else held.pop((m, c))
            for l in reversed(layers):
                act = tape.alloc(layer_size(l)) if rc else None
                tape.free(tape.alloc(align_up(layer_size(l) // 2, cfg.alignment)))
                transients()
                if is_moe(l):
                    inst = f"L{l:02d}.moe.B{m}"
                    if rc:
                        ids = [tape.alloc(moe_size(), inst) for _ in range(MOE_TENSORS_PER_LAYER)]
                        for rid in ids:
                            tape.free(rid, inst)
                    else:
                        for rid in experts.pop((l, m)):
                            tape.free(rid, inst)
                if rc:
                    if prev is not None:
                        tape.free(prev)
                    prev = act
                else:
                    tape.free(acts.pop())
                if m == last_mb:
                    shards.append(tape.alloc(layer_size(l)))
            if rc and prev is not None:
                tape.free(prev)

    tape.begin(PhaseId(PhaseKind.OPTIMIZER))
    for rid in shards:
        tape.free(rid)
    for i in range(2):
        tape.free(tape.alloc(layer_size(i)))
    return tape.finish()


def synth_trace(cfg: SynthConfig) -> Trace:
    """Deterministic synthetic trace (synth.py:263) backed by SoA columns."""
    return Trace.from_arrays(synth_arrays(cfg))


# ---------------------------------------------------------------------------
# pinned benchmark configurations

_L2 = tuple(n * MIB for n in (32, 96, 86, 172))
_MX = tuple(n * MIB for n in (32, 48, 112))
_L3 = tuple(n * MIB for n in (16, 20, 56, 112))
_MOE = dict(num_layers=32, num_microbatches=64, transient_ratio=1.0, size_palette=_MX,
            distinct_sizes=3, persistent_bytes=16384 * MIB, moe_size_range=(4 * MIB, 56 * MIB))
CONFIGS = {
    "c1_llama2_7b_1f1b": ("dense", dict(num_layers=16, num_microbatches=96, transient_ratio=2.0,
                                        size_palette=_L2, distinct_sizes=4, persistent_bytes=8192 * MIB)),
    "c2_llama2_7b_vpp_rcp": ("dense_vpp_recompute", dict(num_layers=32, num_chunks=2, num_microbatches=448,
                                                         transient_ratio=2.0, size_palette=_L2, distinct_sizes=4,
                                                         persistent_bytes=16384 * MIB)),
    "c3_mixtral_moe": ("moe", dict(_MOE)),
    "c3b_mixtral_moe_rcp": ("moe_recompute", dict(_MOE)),
    "c5_llama3_70b": ("dense_vpp_recompute", dict(num_layers=80, num_chunks=4, num_microbatches=1024,
                                                  transient_ratio=4.5, size_palette=_L3, distinct_sizes=4,
                                                  persistent_bytes=20480 * MIB)),
}
C4_PRESETS = ("dense", "dense_recompute", "dense_vpp", "dense_vpp_recompute")
C4_CANDIDATES = ((True, True), (True, False), (False, True), (False, False))


def config(name: str, seed: int = 0) -> SynthConfig:
    preset, kw = CONFIGS[name]
    return SynthConfig.for_preset(preset, seed=seed, **kw)


def c4_config(seed: int) -> SynthConfig:
    """One trace of the batched sweep."""
    return SynthConfig.for_preset(
        C4_PRESETS[seed % 4], seed=seed, num_layers=4 + seed % 29,
        num_microbatches=1 + seed % 8, transient_ratio=0.2 + (seed % 5) * 0.2,
    )
