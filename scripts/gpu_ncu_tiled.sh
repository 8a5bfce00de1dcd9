#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 8 -c 4 -o gpurun_out/prof_tiled python bench.py --steps 2 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > gpurun_out/ncu_tiled.log 2>&1
ls -la gpurun_out
