#!/bin/bash
# GPU-box check with the kernel sweep: -m gpu tests, then the bench line and per-kernel roofline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-configs ${BENCH_ARGS} > gpurun_out/bk.json 2> gpurun_out/bk.err
python - <<'PY' || tail -n 5 gpurun_out/bk.err
import json
d = json.load(open("gpurun_out/bk.json"))
print("bench", round(d["ms_per_step"], 4), "ms/step", round(d["value"] / 1e9, 4), "e9 e2e", round(d["e2e"]["value"] / 1e9, 4))
for k, v in d["kernel_roofline"].items():
    print(" ", k, round(v["ms"], 3), "ms frac", round(v["frac"], 3))
PY
grep -E "passed|failed|error" gpurun_out/tests.log | tail -n 3
