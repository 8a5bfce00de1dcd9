#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-suite --dtype f32 > gpurun_out/bench_f32.json 2> gpurun_out/bench.err
timeout 300 python bench.py --no-suite --no-cpu-baseline > gpurun_out/bench_f64.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --workload liars_dice --no-suite --no-cpu-baseline --dtype f32 > gpurun_out/bench_liars_f32.json 2>> gpurun_out/bench.err
