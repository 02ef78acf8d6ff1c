"""Generate tests/golden/traceio.json from the REFERENCE (run in the build
container, where /root/reference exists): sha256 of the reference's
write_trace output for preset traces, and one reference-planned plan bundle
with the sha256 of its write_plan output.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_traceio_golden.py
"""
import hashlib
import json
import os
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
import memplan as R  # noqa: E402

out = {"trace": {}}
d = tempfile.mkdtemp()
for preset in ("dense", "dense_vpp", "moe", "moe_recompute"):
    tr = R.synth_trace(R.SynthConfig.for_preset(preset, seed=11))
    for form in ("raw", "paired"):
        p = os.path.join(d, "t")
        R.write_trace(tr, p, form=form)
        out["trace"][f"{preset}/11/{form}"] = hashlib.sha256(open(p, "rb").read()).hexdigest()
tr = R.synth_trace(R.SynthConfig.for_preset("moe_recompute", seed=1))
plan, rmap = R.plan_trace(tr)
b = plan.to_bundle(rmap)
p = os.path.join(d, "p")
R.write_plan(b, p)
out["plan_fixture"] = {
    "pool_size": b.pool_size,
    "decisions": [[x.id, x.addr, x.size, x.t_s, x.t_e] for x in b.decisions],
    "reuse": [[list(k), [[iv.lo, iv.hi] for iv in v]] for k, v in b.reuse.items()],
    "sha256": hashlib.sha256(open(p, "rb").read()).hexdigest(),
}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "traceio.json"), "w") as fh:
    json.dump(out, fh, separators=(",", ":"))
print("wrote traceio.json")
