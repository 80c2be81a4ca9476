#!/bin/bash
# Is the one-slice scan at small N limited by the board power cap through the tensor work on
# the padded 128-row slice?  Alternate the product build with ARGUS_SCAN_EXP=2 (one MMA per
# tile instead of 48: scores wrong, diagnostics only) on fixed-N 48 batches, 600 steps.
set -u
OUT=gpurun_out/pwr
mkdir -p $OUT
LIB=paper_2511_06724_b200/libargus.so
python -m paper_2511_06724_b200.build --force > $OUT/build.log 2>&1 || exit 1
cp $LIB /tmp/lib_prod.so
NVCC_EXTRA="-DARGUS_SCAN_EXP=2" python - <<'PY' >> $OUT/build.log 2>&1
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
cp $LIB /tmp/lib_exp2.so
for rep in 1 2 3; do
  for V in prod exp2; do
    cp /tmp/lib_$V.so $LIB; touch $LIB
    timeout 300 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --tensor-n 0 --e2e-steps 2 --fixed-n 48 > $OUT/${V}_$rep.log 2>&1
    nvidia-smi --query-gpu=power.draw,clocks.sm --format=csv,noheader >> $OUT/${V}_$rep.log
  done
done
cp /tmp/lib_prod.so $LIB; touch $LIB
for f in $OUT/*_?.log; do echo "$f $(grep -o '"value": [0-9.]*' $f | head -1) $(grep -o '"hbm_achieved_gbs": [0-9.]*' $f) $(grep -o '"sm_mhz": [0-9.]*' $f)"; done
