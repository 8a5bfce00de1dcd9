#!/bin/bash
# Short perf session: tests, A/B benches.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench.json 2> gpurun_out/bench.err
for wc in 4 8 24; do SCFR_WAVE_CTAS=$wc timeout 600 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench_wc$wc.json 2>> gpurun_out/bench.err; done
timeout 300 python bench.py --workload liars_dice --steps 300 --warmup 5 --no-cpu-baseline --no-suite > gpurun_out/bench_liars.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv --log-file gpurun_out/launches_dram.csv python bench.py --steps 3 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > gpurun_out/ncu_bench.log 2>&1
ls gpurun_out
