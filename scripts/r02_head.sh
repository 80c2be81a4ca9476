#!/bin/bash
# Round 2, restarted session: the GPU suite, smoke and the default C2 line on HEAD.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -m "gpu and not full" -q -p no:cacheprovider > $OUT/pytest_fast.log 2>&1; echo "rc=$?" >> $OUT/pytest_fast.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
for rep in 1 2; do timeout 600 python bench.py > $OUT/bench_C2_$rep.log 2>&1; done
timeout 600 python bench.py --fixed-n 320 --steps 40 --warmup 5 --no-cpu-baseline > $OUT/bench_N320.log 2>&1
tail -3 $OUT/pytest_fast.log; tail -1 $OUT/bench_C2_1.log | cut -c1-400
