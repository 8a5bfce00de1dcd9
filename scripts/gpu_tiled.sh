#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tiled" > gpurun_out/pytest_tiled.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiled.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench_tiled.json 2> gpurun_out/bench_tiled.err
SCFR_ENGINE=1 timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench_levels.json 2>> gpurun_out/bench_tiled.err
timeout 300 python bench.py --workload liars_dice --no-cpu-baseline --no-suite > gpurun_out/bench_liars_tiled.json 2>> gpurun_out/bench_tiled.err
