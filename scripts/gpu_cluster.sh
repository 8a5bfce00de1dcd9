#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for e in 1 5 4; do SCFR_ENGINE=$e timeout 300 python bench.py --workload liars_dice --steps 200 --no-cpu-baseline --no-suite > gpurun_out/bench_liars_e$e.json 2>> gpurun_out/bench.err; done
for e in 0 5; do SCFR_ENGINE=$e timeout 300 python bench.py --workload leduc --steps 200 --no-cpu-baseline --no-suite > gpurun_out/bench_leduc_e$e.json 2>> gpurun_out/bench.err; done
timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench_goof.json 2>> gpurun_out/bench.err
