#!/bin/bash
# GPU tests + create-time probe + default bench (e2e).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python scripts/micro/create_probe.py 2> gpurun_out/cp.log
timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_goof.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_goof2.json 2>> gpurun_out/bench.err
