#!/bin/bash
# DRAM bytes / duration of the multi-slice scans per L2 policy (0 evict-first, 1 normal).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
run() {  # name config fixed_n kernel-regex
  for m in 1 0; do
    ARGUS_SCAN_L2=$m timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:$4 -s 6 -c 2 --csv --log-file $OUT/l2_$1_$m.csv \
      python bench.py --config $2 --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tensor-n 0 --fixed-n $3 > $OUT/l2_$1_$m.log 2>&1
  done
}
run C5 C5 4096 k_scan_pair
run C2n320 C2 320 k_scan_tc
run C2n512 C2 512 k_scan_pair
run C2n1024 C2 1024 k_scan_pair
