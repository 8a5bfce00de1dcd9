#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for f in 0 1; do SCFR_NO_EMPTY_ROWS=$f timeout 300 python bench.py --no-cpu-baseline --no-suite --steps 200 > gpurun_out/bench_goof_noempty$f.json 2>> gpurun_out/bench.err; done
timeout 300 python bench.py --workload liars_dice --no-cpu-baseline --no-suite > gpurun_out/bench_liars.json 2>> gpurun_out/bench.err
