#!/bin/bash
# GPU-box check: bench line (device / e2e), then the -m gpu test summary last.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/tests.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-configs --no-kernel-sweep ${BENCH_ARGS} > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json; d=json.load(open('gpurun_out/b.json')); print('bench', round(d['ms_per_step'],4), 'ms/step', round(d['value']/1e9,4), 'e9', 'e2e', round(d['e2e']['value']/1e9,4))" || tail -n 5 gpurun_out/b.err
grep -E "passed|failed|error" gpurun_out/tests.log | tail -n 3
