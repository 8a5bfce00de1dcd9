#!/bin/bash
# A/B of two builds of the library on one box: $1 = alternative .so (in _lib/).
mkdir -p gpurun_out
L=paper_2605_14277_b200/_lib
cp $L/libseqcfr_b200.so /tmp/main.so
for i in 1 2; do
  cp /tmp/main.so $L/libseqcfr_b200.so
  timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_a$i.json 2>> gpurun_out/bench.err
  cp $L/$1 $L/libseqcfr_b200.so
  timeout 300 python bench.py --no-cpu-baseline --no-suite > gpurun_out/ab_b$i.json 2>> gpurun_out/bench.err
done
cp /tmp/main.so $L/libseqcfr_b200.so
