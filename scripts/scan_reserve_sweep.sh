#!/bin/bash
# ARGUS_SCAN_RESERVE: SMs the pipelined scan leaves free for the next prep / the tail.
mkdir -p gpurun_out
python -m paper_2511_06724_b200.build > gpurun_out/build5.log 2>&1
ARGUS_SCAN_RESERVE=2 timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "pipelined or async or migration" > gpurun_out/rs_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rs_pytest.log
for rep in 1 2; do for rs in 0 2 4; do
  ARGUS_SCAN_RESERVE=$rs timeout 300 python bench.py --no-cpu-baseline > gpurun_out/rs_${rs}_$rep.log 2>&1
  ARGUS_SCAN_RESERVE=$rs timeout 300 python bench.py --no-cpu-baseline --fixed-n 48 --steps 2000 > gpurun_out/rs48_${rs}_$rep.log 2>&1
done; done
