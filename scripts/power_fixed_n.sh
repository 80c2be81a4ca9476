#!/bin/bash
# Sustained-state clocks and rate of the single-slice scan at N = 48 (80 zero-padded
# prompt rows per MMA) against N = 128 (none): does MMA work on padding cost power?
mkdir -p gpurun_out
python -m paper_2511_06724_b200.build > gpurun_out/build4.log 2>&1
for rep in 1 2; do for n in 48 128; do
  timeout 300 python bench.py --no-cpu-baseline --fixed-n $n --steps 2000 --warmup 20 > gpurun_out/pw_n${n}_$rep.log 2>&1
done; done
