#!/bin/bash
# scan variants (diagnostics): two MMA issuers (default) vs one
mkdir -p gpurun_out
python -m paper_2511_06724_b200.build > gpurun_out/sched_build.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "many_tiles or pipelined or ragged" > gpurun_out/sched_pytest.log 2>&1
for v in 2 1; do
  echo "== mma warps=$v" >> gpurun_out/sched_exp.log
  if [ $v = 1 ]; then export ARGUS_SCAN_1MMA=1; fi
  timeout 300 python bench.py --pipeline 0 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 \
     --sweep 64,128,256,384,512,1024 2>&1 | grep sweep >> gpurun_out/sched_exp.log
done
