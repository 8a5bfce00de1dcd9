#!/bin/bash
mkdir -p gpurun_out
SCFR_NO_GRAPH=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python scripts/micro/forest_one.py goof4 pcfr+ alt 3 > gpurun_out/dbg_memcheck_goof4.log 2>&1
SCFR_GROUP_NJ=0 timeout 900 python scripts/forest_check.py --quick --env SCFR_NO_LEAF_FUSE > gpurun_out/lf_check.log 2>&1; echo "rc=$?" >> gpurun_out/lf_check.log
timeout 300 python scripts/micro/timeline.py goof5 20 > gpurun_out/timeline.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep --steps 100 > gpurun_out/bench_lf_$i.json 2>&1
SCFR_NO_LEAF_FUSE=1 timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep --steps 100 > gpurun_out/bench_nolf_$i.json 2>&1
done
