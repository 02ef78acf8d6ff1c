#!/bin/bash
# One `ncu --set full` capture per top kernel of the c4 planner call (tools/one_plan.py).
# usage: bash tools/prof_full.sh <tag> [kernel-regex ...]
tag=${1:-r01}; shift
ks=${@:-k_layers_warp k_seg_bitonic k_validate_tiles k_fusion}
mkdir -p gpurun_out
for k in $ks; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -c 2 \
      -o gpurun_out/${tag}_${k} python tools/one_plan.py > gpurun_out/${tag}_${k}.log 2>&1
  tail -1 gpurun_out/${tag}_${k}.log
done
ls -la gpurun_out
