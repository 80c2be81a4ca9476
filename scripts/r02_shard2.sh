#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not full" -q -x -p no:cacheprovider > $OUT/pytest_fast.log 2>&1; echo "rc=$?" >> $OUT/pytest_fast.log
for G in 8; do
  timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 600 --shard-of $G --force-nccl > $OUT/shard_C2_G$G.log 2>&1
  timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 600 --shard-of $G > $OUT/shard_C2_G${G}_1gpu.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 600 > $OUT/bench_C2.log 2>&1
