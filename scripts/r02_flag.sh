#!/bin/bash
# Prep -> scan through a device flag (ARGUS_SCAN_FLAG) with an early grid trigger: per-CTA
# scan gaps, in-process A/B, GPU tests.
set -u
OUT=gpurun_out/flag
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for F in 0 1; do
  for N in 48 128; do
    ARGUS_SCAN_FLAG=$F timeout 300 python tools/scan_gaps.py --n $N >> $OUT/gaps_f$F.jsonl 2>> $OUT/err.log
  done
done
timeout 300 python tools/ab_env.py ARGUS_SCAN_FLAG 0 1 --n 48 --steps 100 --rounds 8 >> $OUT/ab.jsonl 2>> $OUT/err.log
timeout 400 python tools/ab_env.py ARGUS_SCAN_FLAG 0 1 --n 0 --steps 256 --rounds 6 >> $OUT/ab.jsonl 2>> $OUT/err.log
timeout 900 python -m pytest tests -m "gpu and not full" -q -x -p no:cacheprovider > $OUT/pytest_fast.log 2>&1; echo "rc=$?" >> $OUT/pytest_fast.log
cat $OUT/gaps_f*.jsonl $OUT/ab.jsonl; tail -3 $OUT/pytest_fast.log; tail -5 $OUT/err.log
