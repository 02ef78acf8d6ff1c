"""Live-training integration (paper §4 and §6): the Allocation Profiler that
records a training iteration's raw allocation trace, and the Request Matcher
that tags every CUDA request of a running model with its phase and layer so
the plan can be served.

Both ride on libstw_alloc.so installed as PyTorch's CUDAPluggableAllocator:

    install()                                    # before the first CUDA allocation
    m = RequestMatcher(model, dynamic=[...])     # forward / backward hooks on every module
    ... warm-up iteration (passthrough) ...
    prof = m.profile()                           # record one iteration
    with prof:
        run_iteration(m)                         # uses m.forward(mb) / m.backward(mb) / m.optimizer()
    trace = prof.trace(path)                     # raw JSONL (traceio.py:6-11) -> parse_trace
    plan, rmap = plan_trace(trace)               # on the device
    m.serve(plan.to_bundle(rmap), trace)         # the next iterations run from the plan

Tags: the phase comes from the caller's context managers (init, F:m, B:m, opt:
the reference's PhaseId tags); the layer instance is the innermost running
module, `<module path>.F<mb>` / `.B<mb>` (like the synthetic traces'
`L01.moe.F0`), or `<phase>.step` outside any module; a request is dynamic when
a module named in `dynamic` is on the stack. While serving, static requests
take their planned offsets through the (phase, size) queues and dynamic ones
the reuse key their layer instance recorded, in order.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import json
import os

import numpy as np

from . import _lib
from .domain import DeviceError
from .runtime import ALLOC_PATH, PlanAllocator, load

MODE_PASSTHROUGH, MODE_PROFILE, MODE_SERVE = 0, 1, 2


def _lib_alloc():
    L = load()
    if not getattr(L, "_matcher_types", False):
        L.stw_prof_set.restype = None
        L.stw_prof_records.restype = C.c_int64
        L.stw_set_layer_instance.restype = None
        L._matcher_types = True
    return L


def install():
    """Make libstw_alloc the process's CUDA allocator (passthrough until a plan
    is served); call before the first CUDA allocation."""
    PlanAllocator.install()


class Profile:
    """One recording window of the Allocation Profiler."""

    def __init__(self, matcher: "RequestMatcher"):
        self.m = matcher

    def __enter__(self):
        self.m._profiling = True
        self.m._push()
        if _lib_alloc().stw_alloc_set_mode(MODE_PROFILE) != 0:
            raise DeviceError("cannot enter profiling mode")
        return self

    def __exit__(self, *exc):
        import torch

        torch.cuda.synchronize()
        _lib_alloc().stw_alloc_set_mode(MODE_PASSTHROUGH)
        self.m._profiling = False
        return False

    def records(self) -> dict:
        L = _lib_alloc()
        n = L.stw_prof_records(None, None, None, None, None, None, C.c_int64(0))
        cols = dict(op=np.empty(n, np.int8), dyn=np.empty(n, np.int8), phase=np.empty(n, np.int32),
                    module=np.empty(n, np.int32), id=np.empty(n, np.int64), size=np.empty(n, np.int64))
        L.stw_prof_records(*(_lib.ptr(cols[k]) for k in ("op", "dyn", "phase", "module", "id", "size")),
                           C.c_int64(n))
        return cols

    def write(self, path) -> None:
        """The recording as a raw trace file (traceio.py:6-11: header, then one
        op per line; the line index is the timestamp)."""
        r = self.records()
        phases, modules = self.m._phase_tags, self.m._modules
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(json.dumps({"kind": "trace", "version": 1, "format": "raw"}, sort_keys=True,
                                separators=(",", ":")) + "\n")
            for op, dyn, ph, mod, i, sz in zip(r["op"].tolist(), r["dyn"].tolist(), r["phase"].tolist(),
                                               r["module"].tolist(), r["id"].tolist(), r["size"].tolist()):
                rec = {"op": "alloc" if op == 0 else "free", "id": i, "phase": phases[ph], "module": modules[mod]}
                if op == 0:
                    rec["size"] = sz
                    rec["dynamic"] = bool(dyn)
                fh.write(json.dumps(rec, sort_keys=True, separators=(",", ":")) + "\n")

    def trace(self, path):
        """Write the raw trace and read it back through parse_trace (validated)."""
        from .traceio import parse_trace

        self.write(path)
        return parse_trace(path)


class RequestMatcher:
    """Phase / layer tagging of a running model's CUDA requests (see module doc)."""

    def __init__(self, model, dynamic=()):
        self.model = model
        self.dynamic = set(dynamic)
        self._phase = "init"
        self._mb = 0
        self._stack = []  # (module path, is_dynamic)
        self._profiling = False
        self._phase_tags, self._phase_ix = [], {}
        self._modules, self._module_ix = [], {}
        self._serving = None
        self._handles = []
        for name, mod in model.named_modules():
            if not name:
                continue
            self._handles.append(mod.register_forward_pre_hook(self._enter(name)))
            self._handles.append(mod.register_forward_hook(self._leave()))
            self._handles.append(mod.register_full_backward_pre_hook(self._enter(name)))
            self._handles.append(mod.register_full_backward_hook(self._leave()))

    def detach(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles = []

    # hooks ------------------------------------------------------------------
    def _enter(self, name):
        dyn = name in self.dynamic or any(name.startswith(d + ".") for d in self.dynamic)

        def hook(*_):
            self._stack.append((name, dyn or bool(self._stack and self._stack[-1][1])))
            self._push()

        return hook

    def _leave(self):
        def hook(*_):
            if self._stack:
                self._stack.pop()
            self._push()

        return hook

    def _layer_name(self) -> str:
        suffix = {"F": f"F{self._mb}", "B": f"B{self._mb}"}.get(self._phase[:1], "")
        if self._stack:
            return f"{self._stack[-1][0]}.{suffix}" if suffix else self._stack[-1][0]
        return f"{self._phase}.step"

    def _push(self) -> None:
        dyn = bool(self._stack and self._stack[-1][1])
        L = _lib_alloc()
        if self._profiling:
            ph = self._phase_ix.setdefault(self._phase, len(self._phase_tags))
            if ph == len(self._phase_tags):
                self._phase_tags.append(self._phase)
            name = self._layer_name()
            mi = self._module_ix.setdefault(name, len(self._modules))
            if mi == len(self._modules):
                self._modules.append(name)
            L.stw_prof_set(C.c_int32(ph), C.c_int32(mi), C.c_int32(int(dyn)))
        elif self._serving is not None:
            phase_ix, layer_ix = self._serving
            L.stw_set_phase(C.c_int32(phase_ix.get(self._phase, -1)))
            L.stw_set_layer_instance(C.c_int32(layer_ix.get(self._layer_name(), -1) if dyn else -1),
                                     C.c_int32(int(dyn)))

    # phases -----------------------------------------------------------------
    @contextlib.contextmanager
    def phase(self, tag: str, microbatch: int = 0):
        """Enter a phase. Phases are markers in the op stream, so the phase
        stays current after the block until the next one starts (a raw trace
        may not re-open a phase, traceio.py:112-115)."""
        self._phase, self._mb = tag, microbatch
        self._push()
        yield

    def forward(self, mb: int = 0):
        return self.phase(f"F:{mb}", mb)

    def backward(self, mb: int = 0):
        return self.phase(f"B:{mb}", mb)

    def optimizer(self):
        return self.phase("opt")

    # modes ------------------------------------------------------------------
    def profile(self) -> Profile:
        return Profile(self)

    def serve(self, bundle, trace) -> PlanAllocator:
        """Load the plan (pool reserved in one VA range) and route the next
        requests through it: phase -> schedule index for the static queues,
        layer instance -> its recorded reuse keys for dynamic requests."""
        import torch

        torch.cuda.synchronize()
        rt = PlanAllocator(bundle, trace)  # reserves the pool, loads queues + spaces, enters serving mode
        ta = rt.ta
        names, kidx = ta.dynamic_keys()
        key_pos = {k: i for i, k in enumerate(rt.keys)}
        d = np.nonzero(ta.dyn)[0]
        d = d[np.lexsort((ta.id[d], ta.t_s[d]))]  # recorded (alloc) order
        per_layer = [[] for _ in ta.layer_names]
        for e in d.tolist():
            per_layer[int(ta.ls[e])].append(key_pos.get(names[kidx[e]], -1))
        off = np.zeros(len(per_layer) + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in per_layer])
        keys = np.asarray([k for x in per_layer for k in x], np.int32)
        rc = _lib_alloc().stw_alloc_load_dyn_keys(C.c_int32(len(per_layer)), _lib.ptr(off), _lib.ptr(keys))
        if rc != 0:
            raise DeviceError(f"stw_alloc_load_dyn_keys failed ({rc})")
        phase_ix = {p.tag(): i for i, p in enumerate(ta.phases[:ta.n_sched])}
        layer_ix = {n: i for i, n in enumerate(ta.layer_names)}
        self._serving = (phase_ix, layer_ix)
        self._push()
        return rt


__all__ = ["ALLOC_PATH", "Profile", "RequestMatcher", "install"]
