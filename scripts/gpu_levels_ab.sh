#!/bin/bash
# A/B of the level engine and the tile engine + GPU tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
SCFR_ENGINE=1 timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench_levels.json 2> gpurun_out/bench.err
SCFR_ENGINE=4 timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/bench_tiled.json 2>> gpurun_out/bench.err
SCFR_ENGINE=1 timeout 300 python bench.py --workload liars_dice --no-cpu-baseline --no-suite > gpurun_out/bench_liars_levels.json 2>> gpurun_out/bench.err
SCFR_ENGINE=4 timeout 300 python bench.py --workload liars_dice --no-cpu-baseline --no-suite > gpurun_out/bench_liars_tiled.json 2>> gpurun_out/bench.err
SCFR_ENGINE=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_levels.csv python bench.py --steps 3 --warmup 3 --soak 0 --profile-iters 1 --no-cpu-baseline --no-suite > /dev/null 2>&1
