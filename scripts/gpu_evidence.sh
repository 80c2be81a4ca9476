#!/bin/bash
# Evidence pass: launch list of the bench command, ncu --set full of the scan at
# N=64 and N=256, and the reference arm.  No number from here is a bench value.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 200 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?" >> $OUT/ncu_launches.log
for N in 64 256; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_tc -s 8 -c 1 \
     -o $OUT/prof_scan_N$N -f python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fixed-n $N \
     > $OUT/ncu_full_N$N.log 2>&1
  echo "full N=$N rc=$?" >> $OUT/ncu_full_N$N.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.log 2>&1
echo "reference rc=$?" >> $OUT/bench_reference.log
