#!/bin/bash
# compute-sanitizer over every engine (level engine modes, SMEM / grid /
# cluster persistent engines with their hand-rolled barriers, tile engine).
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/micro/sanitize_cases.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/$tool.log
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
