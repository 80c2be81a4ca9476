#!/bin/bash
# A/B: SM reserve for every pipelined scan (tails of big batches run beside the next scan).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for rep in 1 2 3; do
  timeout 600 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --tensor-n 0 > $OUT/ra0_$rep.log 2>&1
  ARGUS_SCAN_RESERVE_ALL=1 timeout 600 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --tensor-n 0 > $OUT/ra1_$rep.log 2>&1
done
ARGUS_SCAN_RESERVE_ALL=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --tensor-n 0 --fixed-n 320 > $OUT/ra1_f320.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --tensor-n 0 --fixed-n 320 > $OUT/ra0_f320.log 2>&1
