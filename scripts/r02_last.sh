#!/bin/bash
# Last GPU pass of the round on the final commit: the whole GPU suite (the driver's command),
# smoke, and the driver-form bench line.
set -u
OUT=gpurun_out/last
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 1800 python -m pytest tests -x -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_C2_s20.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_reference.log 2>&1
tail -2 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; tail -1 $OUT/bench_C2_s20.log | cut -c1-300
