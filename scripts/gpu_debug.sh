#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/micro/timeline.py goof5 20 > gpurun_out/timeline.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep --steps 100 > gpurun_out/bench_ov.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
