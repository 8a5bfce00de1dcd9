#!/bin/bash
# A/B of library builds on one box with scripts/micro/goof5_ab.py (one
# process per build, alternating): $@ = alternative .so files in _lib/.
L=paper_2605_14277_b200/_lib
cp $L/libseqcfr_b200.so /tmp/main.so
for i in 1 2 3; do
  cp /tmp/main.so $L/libseqcfr_b200.so
  echo -n "main: "; AB_ROUNDS=1 python scripts/micro/goof5_ab.py "" | tail -1
  for alt in "$@"; do
    cp $L/$alt $L/libseqcfr_b200.so
    echo -n "$alt: "; AB_ROUNDS=1 python scripts/micro/goof5_ab.py "" | tail -1
  done
done
cp /tmp/main.so $L/libseqcfr_b200.so
