#!/bin/bash
# k_tail at N = 48 (serial): warp-state samples at the highest sampling rate, per source line.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 ncu --section WarpStateStats --section SourceCounters --warp-sampling-interval 0 \
   --warp-sampling-buffer-size 536870912 --clock-control none --import-source on -k regex:k_tail -s 10 -c 8 \
   -o $OUT/prof_tail_samples_N48 -f python bench.py --steps 6 --warmup 3 --no-cpu-baseline --pipeline 0 --tensor-n 0 \
   --e2e-steps 1 --fixed-n 48 > $OUT/ncu_tail_samples.log 2>&1
tail -3 $OUT/ncu_tail_samples.log
