#!/bin/bash
# Pipelined NCCL path: GPU tests of the one-rank communicator, then C2 / C3 bench lines
# through it (pipelined) next to the single-GPU pipelined lines.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_nccl_path.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest_nccl.log 2>&1
echo "rc=$?" >> $OUT/pytest_nccl.log
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 200 --force-nccl > $OUT/bench_nccl_$rep.log 2>&1
  timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 200 > $OUT/bench_C2_$rep.log 2>&1
done
timeout 600 python bench.py --config C3 --no-cpu-baseline --tensor-n 0 --steps 40 --force-nccl > $OUT/bench_C3_nccl.log 2>&1
timeout 600 python bench.py --config C3 --no-cpu-baseline --tensor-n 0 --steps 40 > $OUT/bench_C3.log 2>&1
