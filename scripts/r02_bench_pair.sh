#!/bin/bash
# C2 bench lines: pipelined (default) and serial (--pipeline 0), 200 steps each, twice alternating.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 200 > $OUT/bench_C2_$rep.log 2>&1
  timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 200 --pipeline 0 > $OUT/bench_serial_$rep.log 2>&1
done
