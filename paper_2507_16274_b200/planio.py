"""Plan files: the reference's single-document JSON layout (traceio.py:334-391).

Byte-identical output to `memplan.write_plan` (canonical `sort_keys`,
`indent=2`, trailing newline) so plan files and their hashes interoperate.
"""

from __future__ import annotations

import json
from pathlib import Path

from .domain import DEFAULT_ALIGNMENT, PlanError
from .ivset import Interval, IntervalSet
from .plan_types import PlanBundle, PlanDecision

SCHEMA_VERSION = 1


def plan_document(bundle: PlanBundle) -> dict:
    cols = getattr(bundle, "_cols", None)
    if cols is not None:
        decs = [{"id": i, "addr": a, "size": s, "t_s": ts, "t_e": te}
                for i, a, s, ts, te in zip(cols.id.tolist(), cols.addr.tolist(), cols.size.tolist(),
                                           cols.t_s.tolist(), cols.t_e.tolist())]
    else:
        decs = [{"id": d.id, "addr": d.addr, "size": d.size, "t_s": d.t_s, "t_e": d.t_e} for d in bundle.decisions]
    return {
        "version": SCHEMA_VERSION,
        "pool_size": bundle.pool_size,
        "alignment": bundle.alignment,
        "decisions": decs,
        "reuse_map": [
            {"l_s": l_s, "l_e": l_e, "intervals": [[iv.lo, iv.hi] for iv in bundle.reuse[(l_s, l_e)]]}
            for (l_s, l_e) in sorted(bundle.reuse)
        ],
    }


def dumps_plan(bundle: PlanBundle) -> str:
    return json.dumps(plan_document(bundle), sort_keys=True, indent=2) + "\n"


def write_plan(bundle: PlanBundle, path) -> None:
    Path(path).write_text(dumps_plan(bundle), encoding="utf-8")


def read_plan(path) -> PlanBundle:
    path = Path(path)
    try:
        doc = json.loads(path.read_text(encoding="utf-8"))
    except json.JSONDecodeError as exc:
        raise PlanError(f"{path}: malformed plan file: {exc}") from None
    if doc.get("version") != SCHEMA_VERSION:
        raise PlanError(f"{path}: unsupported schema version {doc.get('version')}")
    try:
        decisions = tuple(PlanDecision(int(d["id"]), int(d["addr"]), int(d["size"]), int(d["t_s"]), int(d["t_e"]))
                          for d in doc["decisions"])
        reuse = {(str(e["l_s"]), str(e["l_e"])): IntervalSet(Interval(int(lo), int(hi)) for lo, hi in e["intervals"])
                 for e in doc.get("reuse_map", [])}
        bundle = PlanBundle(int(doc["pool_size"]), int(doc.get("alignment", DEFAULT_ALIGNMENT)), decisions, reuse)
    except (KeyError, TypeError, ValueError) as exc:
        raise PlanError(f"{path}: malformed plan file: {exc}") from None
    bundle.validate()
    return bundle
