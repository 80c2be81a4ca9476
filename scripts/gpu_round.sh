#!/bin/bash
# One gpurun session: GPU tests, smoke, bench.  Outputs land in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
{ nvidia-smi; nproc; free -g; lscpu | grep "Model name"; } > $OUT/box.txt 2>&1
python -m paper_2511_06724_b200.build >> $OUT/box.txt 2>&1
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke.log
if [ "${BENCH:-1}" = "1" ]; then
  timeout ${BENCH_TIMEOUT:-900} python bench.py ${BENCH_ARGS:-} > $OUT/bench.log 2>&1
  echo "bench rc=$?" >> $OUT/bench.log
fi
