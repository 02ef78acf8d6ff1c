#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_layers_warp" -c 5 \
    -o gpurun_out/prof_lw python tools/one_plan.py > gpurun_out/ncu_lw.log 2>&1
tail -2 gpurun_out/ncu_lw.log
