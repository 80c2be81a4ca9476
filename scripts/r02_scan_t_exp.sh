#!/bin/bash
# Where the transposed small-N scan loses: product (one-slice k_scan_tc) vs k_scan_t, k_scan_t
# without the column top-k (EXP 1), without the transposed stores too (EXP 2); fixed N = 48.
set -u
OUT=gpurun_out/scantx
mkdir -p $OUT
LIB=paper_2511_06724_b200/libargus.so
python -m paper_2511_06724_b200.build --force > $OUT/build.log 2>&1 || exit 1
cp $LIB /tmp/lib_t0.so
for E in 1 2; do
NVCC_EXTRA="-DARGUS_SCANT_EXP=$E" python - <<'PY' >> $OUT/build.log 2>&1
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
cp $LIB /tmp/lib_t$E.so
done
for rep in 1 2; do
  for V in prod t0 t1 t2; do
    if [ $V = prod ]; then cp /tmp/lib_t0.so $LIB; export ARGUS_SCAN_T=0; else cp /tmp/lib_$V.so $LIB; export ARGUS_SCAN_T=1; fi
    touch $LIB
    timeout 300 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --tensor-n 0 --e2e-steps 2 --fixed-n 48 > $OUT/${V}_$rep.log 2>&1
    timeout 300 python tools/scan_gaps.py --n 48 > $OUT/gaps_${V}_$rep.json 2>> $OUT/err.log
  done
done
cp /tmp/lib_t0.so $LIB; touch $LIB
for f in $OUT/*_?.log; do echo "$f $(grep -o '"value": [0-9.]*' $f | head -1) $(grep -o '"hbm_achieved_gbs": [0-9.]*' $f) $(grep -o '"sm_mhz": [0-9.]*' $f)"; done
cat $OUT/gaps_*.json
