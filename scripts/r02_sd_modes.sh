#!/bin/bash
# Serial dictatorship schedules: GPU suite with windows everywhere and one prompt per step
# everywhere, then the tail phase timestamps per N for both.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
for pp in 0 1024; do
  ARGUS_SD_PP=$pp timeout 1200 python -m pytest tests -m "gpu and not full" -x -q -p no:cacheprovider > $OUT/pytest_sd$pp.log 2>&1; echo "rc=$?" >> $OUT/pytest_sd$pp.log
  tail -2 $OUT/pytest_sd$pp.log
done
NVCC_EXTRA="-DARGUS_TAIL_TIMING=1" python - <<'PY'
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
for pp in 0 1024; do
ARGUS_SD_PP=$pp timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 --pipeline 0 --tensor-n 0 --fixed-n 16 --sweep 48,91,128,192,256,384,512 > $OUT/tail_sd$pp.log 2>&1
done
python -m paper_2511_06724_b200.build --force > /dev/null
