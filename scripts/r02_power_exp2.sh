#!/bin/bash
# How the one-slice scan at N = 48 depends on the tensor work per tile: product build vs
# diagnostics builds (scores wrong) with 1 of 48 MMAs (EXP 2), M = 64 MMAs (EXP 3) and half of
# the k-steps (EXP 4); fixed N = 48, 600 steps, builds alternated.
set -u
OUT=gpurun_out/pwr2
mkdir -p $OUT
LIB=paper_2511_06724_b200/libargus.so
python -m paper_2511_06724_b200.build --force > $OUT/build.log 2>&1 || exit 1
cp $LIB /tmp/lib_prod.so
for E in 2 3 4; do
NVCC_EXTRA="-DARGUS_SCAN_EXP=$E" python - <<'PY' >> $OUT/build.log 2>&1
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
cp $LIB /tmp/lib_exp$E.so
done
for rep in 1 2 3; do
  for V in prod exp2 exp3 exp4; do
    cp /tmp/lib_$V.so $LIB; touch $LIB
    timeout 300 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --tensor-n 0 --e2e-steps 2 --fixed-n 48 > $OUT/${V}_$rep.log 2>&1
  done
done
cp /tmp/lib_prod.so $LIB; touch $LIB
for f in $OUT/*_?.log; do echo "$f $(grep -o '"value": [0-9.]*' $f | head -1) $(grep -o '"hbm_achieved_gbs": [0-9.]*' $f) $(grep -o '"sm_mhz": [0-9.]*' $f)"; done
