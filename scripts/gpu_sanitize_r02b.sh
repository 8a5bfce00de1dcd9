#!/bin/bash
# compute-sanitizer over every engine and mode (incl. the subtree mode and the
# out-of-line SMEM kernel), then the GPU suite.
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/micro/sanitize_cases.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/$tool.log
  tail -3 gpurun_out/sanitizer/$tool.log
done
