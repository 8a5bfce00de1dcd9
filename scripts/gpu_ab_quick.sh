#!/bin/bash
# Quick A/B: GPU tests + Liar's dice and Goofspiel benches (no suite / CPU baseline).
mkdir -p gpurun_out
SKIP=1 #timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --workload liars_dice --no-cpu-baseline --no-suite > gpurun_out/ab_liars.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_goof.json 2>> gpurun_out/bench.err
SCFR_NO_GROUP=0 timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_goof_base.json 2>> gpurun_out/bench.err
