#!/bin/bash
# Fused peer exchange: the NCCL-path tests (now through k_merge_send on the one-rank
# communicator), the two-process external tests, then C2 / C3 through the communicator.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_nccl_path.py tests/test_gpu_two_process.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest_p2p.log 2>&1
echo "rc=$?" >> $OUT/pytest_p2p.log
timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 200 --force-nccl > $OUT/bench_nccl_p2p.log 2>&1
ARGUS_NO_P2P=1 timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 200 --force-nccl > $OUT/bench_nccl_ag.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --tensor-n 0 --steps 200 > $OUT/bench_C2.log 2>&1
