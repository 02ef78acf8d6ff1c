#!/bin/bash
# Round profile bundle (run under gpurun): bench JSON, the ncu launch list of
# the bench step, and one `ncu --set full` capture per hot kernel.
# usage: bash tools/prof_round.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-configs"
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches.csv $B --no-kernel-sweep > gpurun_out/${tag}_launches.log 2>&1
full() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c ${NCU_COUNT:-1} \
      -o gpurun_out/${tag}_${name} "$@" > gpurun_out/${tag}_${name}.log 2>&1
  tail -1 gpurun_out/${tag}_${name}.log
}
NCU_COUNT=2 full k_layers_w32 k_layers_w32 2 python tools/one_plan.py
full k_fusion k_fusion 1 python tools/one_plan.py
NCU_COUNT=2 full k_seg_radix k_seg_radix 2 python tools/one_plan.py
full k_overlap_sweep_c4 k_overlap_sweep 1 python tools/one_plan.py
full k_overlap_sweep_big k_overlap_sweep 7 $B
full k_peak_warp_big k_peak_warp 7 $B
full k_os_pass_big k_os_pass 6 $B
ls -la gpurun_out | tail -30
