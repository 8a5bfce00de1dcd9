#!/bin/bash
# Short session: GPU tests, default bench, create-time trace.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench.json 2> gpurun_out/bench.err
SCFR_TRACE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-suite > /dev/null 2> gpurun_out/create_trace.log
