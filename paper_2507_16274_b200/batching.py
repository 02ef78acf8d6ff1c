"""Concatenate traces into the stw_batch layout (host numpy or device torch)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .soa import TraceArrays

COLS = (("id", np.int64), ("size", np.int64), ("t_s", np.int32), ("t_e", np.int32),
        ("ps", np.int32), ("pe", np.int32), ("dyn", np.uint8))


class HostBatch:
    """Concatenated SoA columns of several traces (host memory)."""

    def __init__(self, traces, pinned: bool = False) -> None:
        traces = list(traces)
        self.traces = traces
        self.T = len(traces)
        counts = np.asarray([len(t) for t in traces], dtype=np.int64)
        self.ev_off = np.zeros(self.T + 1, dtype=np.int64)
        np.cumsum(counts, out=self.ev_off[1:])
        self.N = int(self.ev_off[-1])
        self.horizon = np.asarray([t.horizon for t in traces], dtype=np.int32)
        self.n_sched = np.asarray([t.n_sched for t in traces], dtype=np.int32)
        self.cols = {}
        for name, dt in COLS:
            if self.T == 1:
                arr = np.ascontiguousarray(getattr(traces[0], name), dtype=dt)
            else:
                arr = np.concatenate([np.asarray(getattr(t, name), dtype=dt) for t in traces]) if self.T else np.zeros(0, dt)
            self.cols[name] = arr
        if pinned:
            self.pin()

    def pin(self) -> None:
        """Move columns into page-locked memory (torch pinned tensors)."""
        import torch

        self._pins = {}
        for name, arr in list(self.cols.items()) + [("ev_off", self.ev_off), ("horizon", self.horizon),
                                                    ("n_sched", self.n_sched)]:
            t = torch.from_numpy(arr).pin_memory()
            self._pins[name] = t
            view = t.numpy()
            if name in self.cols:
                self.cols[name] = view
            else:
                setattr(self, name, view)

    @property
    def nbytes(self) -> int:
        return sum(a.nbytes for a in self.cols.values()) + self.ev_off.nbytes + self.horizon.nbytes + self.n_sched.nbytes

    def struct(self) -> _lib.Batch:
        c = self.cols
        return _lib.Batch(self.T, 0, self.N, _lib.ptr(self.ev_off), _lib.ptr(c["id"]), _lib.ptr(c["size"]),
                          _lib.ptr(c["t_s"]), _lib.ptr(c["t_e"]), _lib.ptr(c["ps"]), _lib.ptr(c["pe"]),
                          _lib.ptr(c["dyn"]), _lib.ptr(self.horizon), _lib.ptr(self.n_sched))

    def to_device(self, device="cuda"):
        return DeviceBatch(self, device)


class DeviceBatch:
    """The same columns resident in HBM (torch tensors), for device-side timing."""

    def __init__(self, hb: HostBatch, device="cuda") -> None:
        import torch

        self.T, self.N = hb.T, hb.N
        self.host = hb
        self.t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(device) for k, v in hb.cols.items()}
        self.ev_off = torch.from_numpy(hb.ev_off).to(device)
        self.horizon = torch.from_numpy(hb.horizon).to(device)
        self.n_sched = torch.from_numpy(hb.n_sched).to(device)

    def struct(self) -> _lib.Batch:
        t = self.t
        return _lib.Batch(self.T, 1, self.N, _lib.ptr(self.ev_off), _lib.ptr(t["id"]), _lib.ptr(t["size"]),
                          _lib.ptr(t["t_s"]), _lib.ptr(t["t_e"]), _lib.ptr(t["ps"]), _lib.ptr(t["pe"]),
                          _lib.ptr(t["dyn"]), _lib.ptr(self.horizon), _lib.ptr(self.n_sched))


def single(ta: TraceArrays) -> HostBatch:
    return HostBatch([ta])
