#!/bin/bash
# GPU tests (incl. full-size sampled parity) + one bench line per BASELINE config.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m "${PYTEST_MARK:-gpu}" -x -q ${PYTEST_ARGS:-} --durations=15 > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for C in ${CONFIGS:-C2 C5 C4 C3}; do
  timeout 900 python bench.py --config $C --steps ${STEPS:-100} --warmup 5 ${BENCH_EXTRA:-} > $OUT/bench_$C.log 2>&1
  echo "bench $C rc=$?" >> $OUT/bench_$C.log
done
