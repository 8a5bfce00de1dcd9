#!/bin/bash
# Short perf session: tests, A/B benches.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench.json 2> gpurun_out/bench.err
SCFR_NO_SHAPE=1 timeout 600 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench_noshape.json 2>> gpurun_out/bench.err
SCFR_TRACE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-suite > /dev/null 2> gpurun_out/create_trace.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > gpurun_out/ncu_bench.log 2>&1
ls gpurun_out
