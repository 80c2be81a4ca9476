#!/bin/bash
# ncu --set full of the scan kernel at the given fixed N values
set -u
OUT=gpurun_out
mkdir -p $OUT
for N in ${PNS:-384}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_tc -s 8 -c 1 \
     -o $OUT/prof_scan_N$N -f python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fixed-n $N \
     > $OUT/ncu_full_N$N.log 2>&1
  echo "full N=$N rc=$?" >> $OUT/ncu_full_N$N.log
done
