set -u
OUT=gpurun_out
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/c5_base.json 2>/dev/null
NVCC_EXTRA="-DARGUS_SCAN_EXP=1" python - <<'PY'
import os
from paper_2511_06724_b200 import build as b
b.FLAGS.append(os.environ["NVCC_EXTRA"])
b.build(force=True)
PY
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/c5_exp1.json 2>/dev/null
timeout 300 python bench.py --fixed-n 256 --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/n256_exp1.json 2>/dev/null
python -m paper_2511_06724_b200.build --force > /dev/null
timeout 300 python bench.py --fixed-n 256 --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/n256_base.json 2>/dev/null
python - <<'PY'
import json
for f in ("c5_base","c5_exp1","n256_base","n256_exp1"):
    try:
        j=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, j["roofline"]["scan_ms_per_launch"], j["roofline"]["tensor_tflops_achieved"], j["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
