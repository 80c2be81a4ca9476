#!/bin/bash
# Diagnostics on the GPU box: rebuild the scan with ARGUS_SCAN_EXP=1 (no epilogue
# math) and =2 (one MMA per tile instead of 48), sweep, then restore the product build.
set -u
OUT=gpurun_out
mkdir -p $OUT
for E in 1 2; do
  NVCC_EXTRA="-DARGUS_SCAN_EXP=$E" python - <<'PY'
import os, subprocess
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 --sweep ${SW:-64,128,256,384,512} > $OUT/exp$E.log 2>&1
done
python -m paper_2511_06724_b200.build --force > /dev/null
