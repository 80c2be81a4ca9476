#!/bin/bash
# In-process A/B (tools/ab_env.py) of the SM reserve for pipelined multi-slice scans.
set -u
OUT=gpurun_out/ab
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for R in 4 8; do
  for N in 320 256 512; do
    timeout 300 python tools/ab_env.py ARGUS_SCAN_RESERVE_T 0 $R --n $N --steps 40 --rounds 8 >> $OUT/ab.jsonl 2> $OUT/err_${R}_$N.log
  done
  timeout 400 python tools/ab_env.py ARGUS_SCAN_RESERVE_T 0 $R --n 0 --steps 256 --rounds 6 >> $OUT/ab.jsonl 2> $OUT/err_${R}_c2.log
done
cat $OUT/ab.jsonl
