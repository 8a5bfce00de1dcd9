#!/bin/bash
# Short perf session: tests, PDL on/off, phase trace of the SMEM engine.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/phase_trace.py > gpurun_out/phase_trace.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
SCFR_NO_PDL=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_nopdl.json 2>> gpurun_out/bench.err
for w in liars_dice leduc kuhn; do timeout 300 python bench.py --workload $w --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$w.json 2>> gpurun_out/bench.err; done
SCFR_TRACE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/create_trace.log
ls gpurun_out
