"""The reference domain module's API (`memplan/model.py`): phases, events,
decisions, traces, the error hierarchy, and the peak-live sweep (K1 on the
device, `api.peak_live_bytes`)."""

from .api import clique_lower_bound, peak_live_bytes
from .domain import (
    DEFAULT_ALIGNMENT,
    AllocationDecision,
    LayerSpan,
    MemoryRequestEvent,
    MemplanError,
    PhaseId,
    PhaseKind,
    PhaseSpan,
    PlanError,
    SimulationError,
    Trace,
    TraceError,
    align_up,
)

__all__ = [
    "DEFAULT_ALIGNMENT", "AllocationDecision", "LayerSpan", "MemoryRequestEvent", "MemplanError", "PhaseId",
    "PhaseKind", "PhaseSpan", "PlanError", "SimulationError", "Trace", "TraceError", "align_up",
    "clique_lower_bound", "peak_live_bytes",
]
