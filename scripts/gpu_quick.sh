#!/bin/bash
# Short perf session: tests, phase trace of the SMEM engine, benches.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/phase_trace.py > gpurun_out/phase_trace.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
SCFR_NO_FUSE=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_nofuse.json 2>> gpurun_out/bench.err
for w in liars_dice leduc kuhn; do timeout 300 python bench.py --workload $w --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$w.json 2>> gpurun_out/bench.err; done
ls gpurun_out
