#!/bin/bash
# L2 policy experiment for multi-slice scans (diagnostics)
mkdir -p gpurun_out
python -m paper_2511_06724_b200.build > gpurun_out/l2_build.log 2>&1
for m in 0 1 2; do
  echo "== ARGUS_SCAN_L2=$m" >> gpurun_out/l2_exp.log
  ARGUS_SCAN_L2=$m timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 \
     --sweep 128,256,384,512,1024 2>&1 | grep sweep >> gpurun_out/l2_exp.log
done
