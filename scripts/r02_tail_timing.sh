#!/bin/bash
# Tail phase timestamps only (diagnostics build): serial and pipelined C2 trace batches.
set -u
OUT=gpurun_out
mkdir -p $OUT
NVCC_EXTRA="-DARGUS_TAIL_TIMING=1" python - <<'PY'
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 --pipeline 0 --tensor-n 0 --sweep 48,384 > $OUT/tail_timing_serial.log 2>&1
timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 --pipeline 1 --tensor-n 0 --sweep 48,384 > $OUT/tail_timing_pipe.log 2>&1
python -m paper_2511_06724_b200.build --force > /dev/null
