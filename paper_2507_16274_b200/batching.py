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

    def pack(self) -> bool:
        """Compact copies of id (int32 offsets from the smallest id) and size
        (uint32 multiples of the largest power of two dividing every size) for
        stw_plan_batch(es), which then uploads 25 instead of 33 bytes per event.
        False (nothing changes) when the values do not fit."""
        self._packed = None
        if self.N == 0:
            return False
        ids, sizes = self.cols["id"], self.cols["size"]
        base = int(ids.min())
        if int(ids.max()) - base >= (1 << 31) or int(sizes.min()) <= 0:
            return False
        o = int(np.bitwise_or.reduce(sizes))
        shift = (o & -o).bit_length() - 1
        s32 = sizes >> shift
        if int(s32.max()) >= (1 << 32):
            return False
        id32 = (ids - base).astype(np.int32)
        s32 = s32.astype(np.uint32)
        if getattr(self, "_pins", None) is not None:
            import torch

            id32 = torch.from_numpy(id32).pin_memory().numpy()
            s32 = torch.from_numpy(s32).pin_memory().numpy()
        self._packed = (id32, s32, base, shift)
        return True

    @property
    def upload_nbytes(self) -> int:
        """Bytes stw_plan_batch(es) move host -> device per batch."""
        p = getattr(self, "_packed", None)
        if p is None:
            return self.nbytes
        return self.nbytes - self.cols["id"].nbytes - self.cols["size"].nbytes + p[0].nbytes + p[1].nbytes

    def struct(self) -> _lib.Batch:
        c = self.cols
        b = _lib.Batch(self.T, 0, self.N, _lib.ptr(self.ev_off), _lib.ptr(c["id"]), _lib.ptr(c["size"]),
                       _lib.ptr(c["t_s"]), _lib.ptr(c["t_e"]), _lib.ptr(c["ps"]), _lib.ptr(c["pe"]),
                       _lib.ptr(c["dyn"]), _lib.ptr(self.horizon), _lib.ptr(self.n_sched))
        p = getattr(self, "_packed", None)
        if p is not None:
            b.id32, b.size32, b.id_base, b.size_shift = _lib.ptr(p[0]), _lib.ptr(p[1]), p[2], p[3]
        return b

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
