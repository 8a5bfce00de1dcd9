#!/bin/bash
# Create-time A/B of two builds on one box: $1 = alternative .so (in _lib/);
# scripts/micro/create_probe.py per arm, alternating, 3 rounds.
mkdir -p gpurun_out
L=paper_2605_14277_b200/_lib
cp $L/libseqcfr_b200.so /tmp/main.so
for i in 1 2 3; do
  cp /tmp/main.so $L/libseqcfr_b200.so
  timeout 300 python scripts/micro/create_probe.py 2>> gpurun_out/create_a.log
  cp $L/$1 $L/libseqcfr_b200.so
  timeout 300 python scripts/micro/create_probe.py 2>> gpurun_out/create_b.log
done
cp /tmp/main.so $L/libseqcfr_b200.so
