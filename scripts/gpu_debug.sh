#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/micro/timeline.py goof5 20 > gpurun_out/timeline.log 2>&1
SCFR_TOP_DPS=1000 timeout 300 python scripts/micro/timeline.py goof5 20 > gpurun_out/timeline_ls2.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep --steps 100 > gpurun_out/bench_ls3_$i.json 2>&1
SCFR_TOP_DPS=1000 timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep --steps 100 > gpurun_out/bench_ls2_$i.json 2>&1
done
