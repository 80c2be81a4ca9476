#!/bin/bash
# ncu --set full of k_tail (serial, N = 48 and 384) on the product build; cycle-calibrated timing build.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for N in 48 384; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 10 -c 1 \
   -o $OUT/prof_tail_N$N -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --pipeline 0 --tensor-n 0 \
   --e2e-steps 1 --fixed-n $N > $OUT/ncu_tail_N$N.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --pipeline 0 --tensor-n 0 --steps 200 > $OUT/bench_serial.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 200 > $OUT/bench_C2.log 2>&1
