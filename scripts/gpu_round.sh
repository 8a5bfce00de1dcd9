#!/bin/bash
# One gpurun session: GPU tests, smoke, bench (+ per-game suite), reference
# arm, launch list with DRAM bytes, full ncu captures.  Outputs: gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --dtype f32 --no-cpu-baseline --no-suite > gpurun_out/bench_f32.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --workload liars_dice --no-cpu-baseline --no-suite > gpurun_out/bench_liars.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
SCFR_TRACE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-suite > /dev/null 2> gpurun_out/create_trace.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_dram.csv python bench.py --steps 3 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_level -s 20 -c 10 -o gpurun_out/prof_levels python bench.py --steps 2 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -s 2 -c 1 -o gpurun_out/prof_small python bench.py --workload leduc --steps 20 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > gpurun_out/ncu_small.log 2>&1
ls -la gpurun_out
