#!/bin/bash
# Round 2 first GPU pass: the fast GPU suite, smoke, the default bench line, then the tail probe.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not full" -q -x --durations=10 -p no:cacheprovider > $OUT/pytest_fast.log 2>&1
echo "pytest fast rc=$?" >> $OUT/pytest_fast.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_C2.log 2>&1; echo "rc=$?" >> $OUT/bench_C2.log
bash scripts/r02_tail_probe.sh
