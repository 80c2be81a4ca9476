#!/bin/bash
# Transposed small-N scan (ARGUS_SCAN_T=1): parity first (short timeouts), then A/B.
set -u
OUT=gpurun_out/scant${SUFFIX:-}
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
export ARGUS_SCAN_T=1
timeout 180 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c1 or C1" > $OUT/pytest_c1.log 2>&1; echo "rc=$?" >> $OUT/pytest_c1.log
tail -3 $OUT/pytest_c1.log
if grep -q "rc=0" $OUT/pytest_c1.log; then
  timeout 900 python -m pytest tests -m "gpu and not full" -q -p no:cacheprovider > $OUT/pytest_fast.log 2>&1; echo "rc=$?" >> $OUT/pytest_fast.log
  tail -3 $OUT/pytest_fast.log
  unset ARGUS_SCAN_T
  for N in 48 16 64; do
    timeout 300 python tools/ab_env.py ARGUS_SCAN_T 0 1 --n $N --steps 200 --rounds 8 >> $OUT/ab.jsonl 2>> $OUT/err.log
  done
  timeout 400 python tools/ab_env.py ARGUS_SCAN_T 0 1 --n 0 --steps 256 --rounds 12 >> $OUT/ab.jsonl 2>> $OUT/err.log
  cat $OUT/ab.jsonl; tail -3 $OUT/err.log
fi
