#!/bin/bash
# Final bench lines with the final bench.py (config split, e2e after the ramp).
set -u
OUT=gpurun_out/fb
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || exit 1
for rep in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_C2_s20_$rep.log 2>&1
  timeout 600 python bench.py --steps 600 --warmup 5 --no-cpu-baseline > $OUT/bench_C2_s600_$rep.log 2>&1
done
for C in C3 C4 C5; do timeout 600 python bench.py --config $C --steps 40 --warmup 5 --no-cpu-baseline > $OUT/bench_$C.log 2>&1; done
for f in $OUT/bench_*.log; do tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$f', d['value'], d['e2e']['value'], d['e2e']['sync_call_prompts_per_s'], r['bound'], r['frac'], d['clocks']['sm_mhz'], (d.get('tensor_regime') or {}).get('frac'))"; done
