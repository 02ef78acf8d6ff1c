tag=$1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-configs --no-kernel-sweep"
timeout 900 ncu --nvtx --nvtx-include "bench_step/" \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches.csv $B > gpurun_out/${tag}_launches.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "bench_step/" --cache-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    --csv --log-file gpurun_out/${tag}_launches_warm.csv $B > gpurun_out/${tag}_launches_warm.log 2>&1
