"""B200-native STWeaver planner + replay scorer: a drop-in for the reference
`memplan` API (`memplan/__init__.py:1-47`).

    import paper_2507_16274_b200 as memplan
    plan, rmap = memplan.plan_trace(trace)
    report, log = memplan.simulate(trace, plan.to_bundle(rmap))

The reference's module paths work too (`paper_2507_16274_b200.planner`,
`.sim`, `.reuse`, `.baseline`, `.model`, `.intervals`, `.traceio`, `.synth`),
sub-operations included (`pack_group`, `try_fuse`, `build_layers_for_size`,
`CachingAllocator`, `dynamic_allocate`, `compute_metrics`, ...).

Every planning / validation / reuse / replay call runs hand-written sm_100a
CUDA through libstw.so (include/stw.h); there is no CPU fallback.
"""

from .domain import (
    DEFAULT_ALIGNMENT,
    AllocationDecision,
    DeviceError,
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
from .ivset import Interval, IntervalSet, best_fit, intersect, subtract
from .plan_types import (
    MemoryLayer,
    PlanBundle,
    PlanDecision,
    PlanStats,
    ReuseEntry,
    ReuseMap,
    SimReport,
    StaticPlan,
)
from .api import (
    clique_lower_bound,
    compute_reusable_space,
    derive_reuse_map,
    group_dynamic,
    peak_live_bytes,
    plan_batch,
    plan_trace,
    run_baseline,
    simulate,
    synthesize_static_plan,
    validate_plan,
)
from .planner import (
    HomoPhaseGroup,
    LocalPlan,
    build_layers_for_size,
    compute_tmp,
    fuse_plans,
    group_by_phase,
    pack_group,
    try_fuse,
    weighted_tmp_average,
)
from .baseline import CachingAllocator
from .sim import PoolState, compute_metrics, dynamic_allocate
from .traceio import parse_trace, read_plan, write_plan, write_trace
from .tracegen import PRESETS, SynthConfig, SynthConfigError, synth_trace

__version__ = "0.1.0"
