#!/bin/bash
# Quick A/B: GPU tests + Liar's dice and Goofspiel benches (no suite / CPU
# baseline); the third line is the Goofspiel bench with $1 (VAR=value) set.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --workload liars_dice --no-cpu-baseline --no-suite > gpurun_out/ab_liars.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_goof.json 2>> gpurun_out/bench.err
env ${1:-SCFR_NONE=0} timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_goof_base.json 2>> gpurun_out/bench.err
