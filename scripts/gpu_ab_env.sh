#!/bin/bash
# Alternating A/B of one env switch on the default bench: $1 = VAR=value for the B arm.
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_a$i.json 2>> gpurun_out/bench.err
  env $1 timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_b$i.json 2>> gpurun_out/bench.err
done
