#!/bin/bash
# Forest mode: bit-equality against the plain level engine, then the default
# bench with forest on and off on the same box.
mkdir -p gpurun_out
timeout 900 python scripts/forest_check.py > gpurun_out/forest_check.log 2>&1; echo "rc=$?" >> gpurun_out/forest_check.log
timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep > gpurun_out/bench_forest.json 2> gpurun_out/bench_forest.err
SCFR_NO_FOREST=1 timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep > gpurun_out/bench_noforest.json 2> gpurun_out/bench_noforest.err
