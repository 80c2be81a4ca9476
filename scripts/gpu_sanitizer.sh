#!/bin/bash
# compute-sanitizer over the GPU parity tests on the current kernels (profiles/sanitizer/).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build_san.log 2>&1 || { cat $OUT/build_san.log; exit 1; }
timeout 1200 compute-sanitizer --tool memcheck --target-processes all python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_parity.py tests/test_gpu_control.py tests/test_gpu_lifecycle.py tests/test_gpu_nccl_path.py \
  > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 900 compute-sanitizer --tool synccheck --target-processes all python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_parity.py -k "c1_parity or many_tiles or wide_and_narrow" > $OUT/synccheck.log 2>&1; echo "rc=$?" >> $OUT/synccheck.log
