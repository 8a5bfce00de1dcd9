#!/bin/bash
# Forest mode: launch list (per-kernel time + DRAM bytes) and one full capture
# of the OBS forest kernel and the PRED top kernel.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 120 --csv --log-file gpurun_out/forest_launches.csv python bench.py --steps 3 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite --no-sweep > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forest|k_top" -s 16 -c 8 -o gpurun_out/prof_forest python bench.py --steps 2 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite --no-sweep > gpurun_out/ncu_full.log 2>&1
