#!/bin/bash
# A/B of the scan's L2 prefetch of its first chunk: sweep (fixed N) + C2 shard 8 + C2, twice.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not full" -q -x -p no:cacheprovider > $OUT/pytest_fast.log 2>&1; echo "rc=$?" >> $OUT/pytest_fast.log
for rep in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --tensor-n 0 --sweep 16,48,128,320 > $OUT/pf_sweep_$rep.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 600 --shard-of 8 > $OUT/pf_shard8_$rep.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 600 > $OUT/pf_C2_$rep.log 2>&1
done
