"""`memplan` import name for this package, so code (and test files) written
against the reference's module paths run unchanged on libstw:

    PYTHONPATH=tools/memplan_shim:. python -c "import memplan; print(memplan.plan_trace)"

Every `memplan.<module>` resolves to `paper_2507_16274_b200.<module>`.
"""

import importlib
import sys

_pkg = importlib.import_module("paper_2507_16274_b200")
for _sub in ("model", "intervals", "planner", "reuse", "sim", "baseline", "traceio", "synth"):
    sys.modules[f"{__name__}.{_sub}"] = importlib.import_module(f"paper_2507_16274_b200.{_sub}")
sys.modules[__name__] = _pkg
