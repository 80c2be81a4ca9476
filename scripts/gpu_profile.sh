#!/bin/bash
# ncu evidence for the bench workload: launch list (cold, serialised) + one full
# capture of the scan kernel.  Never a bench number.
set -u
OUT=gpurun_out
mkdir -p $OUT
ARGS="--steps ${PSTEPS:-20} --warmup 3 --no-cpu-baseline --e2e-steps 2 ${PEXTRA:-}"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${PCOUNT:-300} --csv \
   --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?" >> $OUT/ncu_launches.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${PKERNEL:-k_scan_tc} -s ${PSKIP:-6} -c ${PCAP:-2} \
   -o $OUT/prof_scan -f python bench.py $ARGS > $OUT/ncu_full.log 2>&1
echo "full rc=$?" >> $OUT/ncu_full.log
