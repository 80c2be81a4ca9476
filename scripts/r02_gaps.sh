#!/bin/bash
# Per-CTA timestamps of consecutive one-slice scans (tools/scan_gaps.py).
set -u
OUT=gpurun_out/gaps
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for N in 48 128; do
  for P in 1 0; do
    timeout 300 python tools/scan_gaps.py --n $N --pipeline $P >> $OUT/gaps.jsonl 2>> $OUT/err.log
  done
done
cat $OUT/gaps.jsonl; tail -5 $OUT/err.log
