#!/bin/bash
# Fast GPU tests first, then full-size tests, then the requested bench configs.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not full" -q -x --durations=10 -p no:cacheprovider > $OUT/pytest_fast.log 2>&1
echo "pytest fast rc=$?" >> $OUT/pytest_fast.log
if [ "${FULL:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m "full" -q --durations=10 -p no:cacheprovider > $OUT/pytest_full.log 2>&1
  echo "pytest full rc=$?" >> $OUT/pytest_full.log
fi
for C in ${CONFIGS:-}; do
  timeout 600 python bench.py --config $C --steps ${STEPS:-100} --warmup 5 ${BENCH_EXTRA:-} > $OUT/bench_$C.log 2>&1
  echo "bench $C rc=$?" >> $OUT/bench_$C.log
done
