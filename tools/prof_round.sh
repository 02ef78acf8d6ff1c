#!/bin/bash
# Round profile bundle (run under gpurun, one GPU): the bench line, the ncu
# launch list of the bench step, and one `ncu --set full` capture per hot
# kernel -- each taken on the SAME launch bench.py times, selected by the NVTX
# ranges bench.py opens (bench_step/ around a timed step; sweep_<kernel>/
# around the >> L2 roofline launches).
# usage: bash tools/prof_round.sh <tag>;  then python tools/make_profile_summary.py <tag>
tag=${1:-r02}
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-configs"
timeout 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 ncu --nvtx --nvtx-include "bench_step/" \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches.csv $B --no-kernel-sweep > gpurun_out/${tag}_launches.log 2>&1
# the same launch list without ncu's cache flush between kernels: the DRAM
# bytes each kernel really moves inside the pipelined call (L2-resident
# intermediates are not re-read from HBM)
timeout 900 ncu --nvtx --nvtx-include "bench_step/" --cache-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches_warm.csv $B --no-kernel-sweep > gpurun_out/${tag}_launches_warm.log 2>&1
full() {  # name nvtx-range kernel-regex count [extra bench args]
  local name=$1 range=$2 rx=$3 cnt=$4; shift 4
  timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$range" \
      -k regex:"$rx" -c $cnt -o gpurun_out/${tag}_${name} $B "$@" > gpurun_out/${tag}_${name}.log 2>&1
  echo "$name: $(tail -1 gpurun_out/${tag}_${name}.log)"
}
full k_layers_w32 "bench_step/" '^k_layers_w32' 2 --no-kernel-sweep
full k_fusion "bench_step/" '^k_fusion$' 1 --no-kernel-sweep
full k_items_sorted "bench_step/" 'k_items_sorted' 1 --no-kernel-sweep
full k_overlap_sweep_c4 "bench_step/" 'k_overlap_sweep' 1 --no-kernel-sweep
full k_peak_warp_big "sweep_k_peak_warp/" 'k_peak_warp' 1
full k_overlap_sweep_big "sweep_k_overlap_sweep/" 'k_overlap_sweep' 1
full k_os_pass_big "sweep_radix_sort_pairs/" 'k_os_pass' 1
full k_os_hist_big "sweep_radix_sort_pairs/" 'k_os_hist' 1
full k_scan_lb_big "sweep_k_scan_lb/" 'k_scan_lb' 1
# the sequential replay warp (c1 baseline) and the whole-GPU layer kernel (c5)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_replay_reg -c 1 \
    -o gpurun_out/${tag}_k_replay_reg_c1 python tools/one_replay.py c1_llama2_7b_1f1b baseline \
    > gpurun_out/${tag}_k_replay_reg_c1.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_layers_big -c 1 \
    -o gpurun_out/${tag}_k_layers_big_c5 python tools/c5_plan_once.py > gpurun_out/${tag}_k_layers_big_c5.log 2>&1
ls -la gpurun_out | grep "$tag" | tail -30
