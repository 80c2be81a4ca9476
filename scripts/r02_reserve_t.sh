#!/bin/bash
# A/B: SM reserve for pipelined multi-slice (tensor-bound) scans, so the previous batch's
# tail runs beside the scan instead of after it (ARGUS_SCAN_RESERVE_T).
set -u
OUT=gpurun_out/rt
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for rep in 1 2; do
for R in 0 3 5 8; do
  for N in 256 320 512; do
    ARGUS_SCAN_RESERVE_T=$R timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --tensor-n 0 --e2e-steps 2 --fixed-n $N > $OUT/r${R}_n${N}_$rep.log 2>&1
  done
  ARGUS_SCAN_RESERVE_T=$R timeout 600 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --tensor-n 0 --e2e-steps 2 > $OUT/r${R}_c2_$rep.log 2>&1
done
done
