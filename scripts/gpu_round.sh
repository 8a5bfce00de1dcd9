#!/bin/bash
# One gpurun session: GPU tests, smoke, benches for every workload, launch
# list and full ncu captures.  Outputs: gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for w in leduc liars_dice kuhn; do timeout 300 python bench.py --workload $w --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$w.json 2>> gpurun_out/bench.err; done
SCFR_NO_SMEM=1 timeout 300 python bench.py --workload leduc --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/bench_leduc_nosmem.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_small -s 3 -c 1 -o gpurun_out/prof_leduc_small python bench.py --workload leduc --steps 20 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline > gpurun_out/ncu_full_leduc.log 2>&1
ls -la gpurun_out
