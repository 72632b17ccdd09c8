#!/bin/bash
# compute-sanitizer pass over every kernel family (run under gpurun, one GPU).
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  mode=""
  [ "$tool" = "racecheck" ] && mode="quick"
  timeout 1200 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py $mode > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
