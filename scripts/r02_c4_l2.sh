#!/bin/bash
# C4 scan DRAM bytes and duration per L2 policy of the cache stream (ARGUS_SCAN_L2=0 evict-first,
# 1 normal (default for several slices), 2 evict-last).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for m in 1 2 0; do
  ARGUS_SCAN_L2=$m timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:k_scan_pair -s 3 -c 2 --csv --log-file $OUT/c4_l2_$m.csv \
    python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 --tensor-n 0 > $OUT/c4_l2_$m.log 2>&1
done
