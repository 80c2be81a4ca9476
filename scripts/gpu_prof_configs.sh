#!/bin/bash
# ncu --set full of one scan launch per config (tensor-bound C5 / C4, HBM-bound C2 N=64).
# No number from here is a bench value.
set -u
OUT=gpurun_out
mkdir -p $OUT
for spec in ${PROF_SPECS:-"C5:4096" "C4:8192"}; do
  C=${spec%%:*}; N=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_tc -s 6 -c 1 \
     -o $OUT/prof_scan_${C}_N$N -f python bench.py --config $C --steps 4 --warmup 3 --no-cpu-baseline \
     --e2e-steps 1 --fixed-n $N > $OUT/ncu_${C}_N$N.log 2>&1
  echo "ncu $C N=$N rc=$?" >> $OUT/ncu_${C}_N$N.log
done
