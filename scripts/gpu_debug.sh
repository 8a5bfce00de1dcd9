#!/bin/bash
mkdir -p gpurun_out
SCFR_GROUP_NJ=0 timeout 900 python scripts/mode_check.py --quick --env SCFR_NO_LEAF_FUSE > gpurun_out/lf_check.log 2>&1; echo "rc=$?" >> gpurun_out/lf_check.log
timeout 300 python scripts/micro/timeline.py goof5 20 > gpurun_out/timeline.log 2>&1
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep --steps 100 > gpurun_out/bench_pf_$i.json 2>&1; done
