#!/bin/bash
# Level merge A/B (Liar's dice, Goofspiel, per-game suite) + GPU tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for m in 0 1; do
  SCFR_NO_LEVEL_MERGE=$m timeout 300 python bench.py --workload liars_dice --no-cpu-baseline --no-suite > gpurun_out/bench_liars_m$m.json 2>> gpurun_out/bench.err
  SCFR_NO_LEVEL_MERGE=$m timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_goof_m$m.json 2>> gpurun_out/bench.err
done
