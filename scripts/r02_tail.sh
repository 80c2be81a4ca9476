#!/bin/bash
# Tail rework check: fast GPU suite, tail phase timestamps (serial), serial + pipelined bench lines.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
export ARGUS_PARITY_REPORT=$OUT/parity_report.jsonl
rm -f $ARGUS_PARITY_REPORT
timeout 900 python -m pytest tests -m "gpu and not full" -q -x -p no:cacheprovider > $OUT/pytest_fast.log 2>&1
echo "pytest fast rc=$?" >> $OUT/pytest_fast.log
NVCC_EXTRA="-DARGUS_TAIL_TIMING=1" python - <<'PY'
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 --pipeline 0 --tensor-n 0 --sweep 16,48,96,384,512 > $OUT/tail_timing_serial.log 2>&1
timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 --pipeline 1 --tensor-n 0 --sweep 48,384 > $OUT/tail_timing_pipe.log 2>&1
python -m paper_2511_06724_b200.build --force > /dev/null
timeout 600 python bench.py --no-cpu-baseline --pipeline 0 --tensor-n 0 > $OUT/bench_serial.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_C2.log 2>&1
