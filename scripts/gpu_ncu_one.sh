#!/bin/bash
mkdir -p gpurun_out
SCFR_ENGINE=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_level<.int.[34], .int.1, .bool.0>" -s 4 -c 2 -o gpurun_out/prof_ilp python bench.py --steps 2 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > gpurun_out/ncu_ilp.log 2>&1
