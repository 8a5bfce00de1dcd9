#!/bin/bash
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_level -s 25 -c 25 -o gpurun_out/prof_iter python bench.py --steps 2 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > gpurun_out/ncu_iter.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_dram.csv python bench.py --steps 3 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out
