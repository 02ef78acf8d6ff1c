#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: memcheck, racecheck (shared-memory
# hazards), synccheck (barrier misuse); summaries into gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 python tools/sanitize_run.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload ok' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
