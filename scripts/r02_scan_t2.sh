#!/bin/bash
# k_scan_t with the row-layout epilogue: its parity tests, then A/B against k_scan_tc.
set -u
OUT=gpurun_out/scant${SUFFIX:-2}
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_scan_t.py -x -q -p no:cacheprovider > $OUT/pytest_scan_t.log 2>&1; echo "rc=$?" >> $OUT/pytest_scan_t.log
tail -3 $OUT/pytest_scan_t.log
if grep -q "rc=0" $OUT/pytest_scan_t.log; then
  for N in 48 16 64; do
    timeout 300 python tools/ab_env.py ARGUS_SCAN_T 0 1 --n $N --steps 200 --rounds 8 >> $OUT/ab.jsonl 2>> $OUT/err.log
  done
  timeout 400 python tools/ab_env.py ARGUS_SCAN_T 0 1 --n 0 --steps 256 --rounds 12 >> $OUT/ab.jsonl 2>> $OUT/err.log
  for rep in 1 2; do for T in 0 1; do
    ARGUS_SCAN_T=$T timeout 300 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --tensor-n 0 --e2e-steps 2 --fixed-n 48 > $OUT/bench_t${T}_$rep.log 2>&1
  done; done
  cat $OUT/ab.jsonl; tail -3 $OUT/err.log
  for f in $OUT/bench_*.log; do echo "$f $(grep -o '"value": [0-9.]*' $f | head -1) $(grep -o '"hbm_achieved_gbs": [0-9.]*' $f) $(grep -o '"sm_mhz": [0-9.]*' $f)"; done
fi
