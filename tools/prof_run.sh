#!/bin/bash
# GPU-box profiling recipe (B200_PROFILING.md): launch list + full capture of the top kernels.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_layers_warp|k_validate_tiles|k_radix_scatter|k_fusion" \
    -s 40 -c 8 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
