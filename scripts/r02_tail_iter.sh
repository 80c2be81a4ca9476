#!/bin/bash
# Tail iteration: GPU parity suite (fast), then the phase timestamps (diagnostics build) at
# N = 16 / 48 / 91 / 384 serial, then sync-call costs on the product build.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -m "gpu and not full" -x -q -p no:cacheprovider > $OUT/pytest_iter.log 2>&1; echo "rc=$?" >> $OUT/pytest_iter.log
tail -3 $OUT/pytest_iter.log
NVCC_EXTRA="-DARGUS_TAIL_TIMING=1" python - <<'PY'
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 --pipeline 0 --tensor-n 0 --sweep 16,48,91,384 > $OUT/tail_timing_serial.log 2>&1
python -m paper_2511_06724_b200.build --force > /dev/null
timeout 600 python tools/sync_cost.py > $OUT/sync_cost.txt 2>&1
