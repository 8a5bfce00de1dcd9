#!/bin/bash
mkdir -p gpurun_out
SCFR_NO_GRAPH=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python scripts/micro/forest_one.py goof4 pcfr+ alt 3 > gpurun_out/dbg_memcheck_goof4.log 2>&1
timeout 900 python scripts/forest_check.py --quick > gpurun_out/top_check.log 2>&1; echo "rc=$?" >> gpurun_out/top_check.log
timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep > gpurun_out/bench_top.json 2> gpurun_out/bench_top.err
SCFR_NO_TOP=1 timeout 300 python bench.py --no-cpu-baseline --no-suite --no-sweep > gpurun_out/bench_notop.json 2> gpurun_out/bench_notop.err
