#!/bin/bash
# --steps 20 (the driver's form) against --steps 600, alternating, three times.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for rep in 1 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --tensor-n 0 > $OUT/st20_$rep.log 2>&1
  timeout 600 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --tensor-n 0 > $OUT/st600_$rep.log 2>&1
done
