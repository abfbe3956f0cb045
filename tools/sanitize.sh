#!/bin/bash
# compute-sanitizer evidence (run under gpurun): racecheck, synccheck, memcheck over
# tools/sanitize_cases.py; logs go to gpurun_out/ (summaries copied to profiles/ by hand)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py \
    > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02_sanitize_$tool.log
  tail -3 gpurun_out/r02_sanitize_$tool.log
done
