#!/bin/bash
# Synchronous host call cost breakdown + the driver-form bench line after the config split.
set -u
OUT=gpurun_out/sync
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 600 python tools/sync_cost.py > $OUT/sync_cost.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_s20.log 2>&1
cat $OUT/sync_cost.txt; tail -1 $OUT/bench_s20.log | cut -c1-1500
