#!/bin/bash
# Per-N scan rates on the C2 cache (the bursty trace's sizes and beyond) and an ncu
# --set full capture of the three-slice scan at N = 320.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --tensor-n 0 \
   --sweep 16,32,48,64,96,128,160,192,256,288,320,352,384,448,512,1024,2048,4096 > $OUT/sweep_C2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_tc -s 6 -c 1 \
   -o $OUT/prof_C2_N320 -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tensor-n 0 \
   --fixed-n 320 > $OUT/ncu_C2_N320.log 2>&1
