#!/bin/bash
# compute-sanitizer on the round-2 kernels (rebuilt tail, k_merge_send, bf16 prep, score capture).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build_san.log 2>&1 || { cat $OUT/build_san.log; exit 1; }
timeout 1500 compute-sanitizer --tool memcheck --target-processes all python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_parity.py tests/test_gpu_parity_exact.py tests/test_gpu_control.py tests/test_gpu_lifecycle.py \
  tests/test_gpu_nccl_path.py -m "gpu and not full" > $OUT/memcheck_r02.log 2>&1; echo "rc=$?" >> $OUT/memcheck_r02.log
timeout 900 compute-sanitizer --tool synccheck --target-processes all python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_parity.py tests/test_gpu_parity_exact.py -k "c1_parity or t2_exact or bf16" > $OUT/synccheck_r02.log 2>&1; echo "rc=$?" >> $OUT/synccheck_r02.log
timeout 900 compute-sanitizer --tool racecheck --target-processes all python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_parity.py -k "c1_parity or ragged_parity" > $OUT/racecheck_r02.log 2>&1; echo "rc=$?" >> $OUT/racecheck_r02.log
