#!/bin/bash
# k_scan_t vs k_scan_tc on the C2 trace, separate processes alternated (600 steps each).
set -u
OUT=gpurun_out/scantc2
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || exit 1
for rep in 1 2 3 4; do for T in 0 1; do
  ARGUS_SCAN_T=$T timeout 300 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --tensor-n 0 --e2e-steps 2 > $OUT/c2_t${T}_$rep.log 2>&1
done; done
for f in $OUT/c2_*.log; do echo "$f $(grep -o '"value": [0-9.]*' $f | head -1) $(grep -o '"sm_mhz": [0-9.]*' $f)"; done
