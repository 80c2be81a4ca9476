#!/bin/bash
# Round 2 diagnostics: phase timestamps of the fused tail (device printf build) in
# serial and pipelined mode, then an ncu --set full capture of k_tail (product build).
set -u
OUT=gpurun_out
mkdir -p $OUT
NVCC_EXTRA="-DARGUS_TAIL_TIMING=1" python - <<'PY'
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 --pipeline 0 --sweep 16,48,96,384,512 > $OUT/tail_timing_serial.log 2>&1
timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 1 --pipeline 1 --sweep 16,48,384 > $OUT/tail_timing_pipe.log 2>&1
python -m paper_2511_06724_b200.build --force > /dev/null
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --pipeline 0 --sweep 16,48,96,384,512 > $OUT/bench_serial.log 2>&1
for N in 48 384; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 10 -c 1 \
   -o $OUT/prof_tail_N$N -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --pipeline 0 \
   --e2e-steps 1 --fixed-n $N > $OUT/ncu_tail_N$N.log 2>&1
done
