#!/bin/bash
cp paper_2605_14277_b200/_lib/libseqcfr_b200.so /tmp/cur.so
for v in head B C cur; do
  if [ $v = cur ]; then cp /tmp/cur.so paper_2605_14277_b200/_lib/libseqcfr_b200.so; else cp scripts/micro/bis/$v/libseqcfr_b200.so paper_2605_14277_b200/_lib/libseqcfr_b200.so; fi
  echo "== $v"; MALLOC_CHECK_=3 timeout 120 python scripts/micro/abort_probe.py 2>&1 | grep -v "^  File" | tail -2
done
