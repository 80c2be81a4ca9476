#!/bin/bash
# Diagnostics: phase timestamps of the fused tail (device printf), then restore the product build.
mkdir -p gpurun_out
NVCC_EXTRA="-DARGUS_TAIL_TIMING=1" python - <<'PY'
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 --sweep 16,96,384 > gpurun_out/tail_timing.log 2>&1
python -m paper_2511_06724_b200.build --force > /dev/null
