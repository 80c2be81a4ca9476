#!/bin/bash
# Per-GPU bound at G GPUs: C2 / C3 with one GPU's stripe (M / G) through the one-rank NCCL
# path (pipelined, fused exchange), and the plain single-GPU pipelined path for reference.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for G in 2 4 8; do
  timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 600 --shard-of $G --force-nccl > $OUT/shard_C2_G$G.log 2>&1
  timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 600 --shard-of $G > $OUT/shard_C2_G${G}_1gpu.log 2>&1
  timeout 900 python bench.py --config C3 --no-cpu-baseline --tensor-n 0 --steps 80 --shard-of $G --force-nccl > $OUT/shard_C3_G$G.log 2>&1
done
