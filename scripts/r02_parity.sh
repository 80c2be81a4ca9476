#!/bin/bash
# Round 2 parity additions: T2 replays, striped T2, -0, odd N*k, G = 1..8, two processes.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
export ARGUS_PARITY_REPORT=$OUT/parity_report.jsonl
rm -f $ARGUS_PARITY_REPORT
timeout 1500 python -m pytest tests/test_gpu_parity_exact.py tests/test_gpu_two_process.py tests/test_gpu_parity.py \
   -m gpu -q -rA --durations=15 -p no:cacheprovider > $OUT/pytest_parity.log 2>&1
echo "rc=$?" >> $OUT/pytest_parity.log
