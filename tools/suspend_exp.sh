#!/bin/bash
# Diagnostics: mbarrier try_wait with a suspend-time hint (ARGUS_MBAR_SUSPEND_NS) vs the
# product build, on the tensor-bound pair scan (N = 256 and C5).  Restores the product build.
set -u
OUT=gpurun_out
mkdir -p $OUT
run() {
  for i in 1 2; do
    timeout 300 python bench.py --fixed-n 256 --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/sus_$1_n256_$i.json 2>/dev/null
  done
  timeout 300 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/sus_$1_c5.json 2>/dev/null
}
run base
for NS in ${NS_LIST:-20000 1000000}; do
  NVCC_EXTRA="-DARGUS_MBAR_SUSPEND_NS=$NS" python - <<'PY'
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
  run $NS
done
python -m paper_2511_06724_b200.build --force > /dev/null
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/sus_*.json")):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, j["roofline"]["scan_ms_per_launch"], j["roofline"]["tensor_tflops_achieved"], j["clocks"]["sm_mhz"])
    except Exception as e:
        print(f, "ERR", e)
PY
