#!/bin/bash
mkdir -p gpurun_out
python -m paper_2511_06724_b200.build > gpurun_out/build7.log 2>&1
timeout 1200 python -m pytest tests -m full -q > gpurun_out/rf_pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/rf_pytest_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 200 --csv \
   --log-file gpurun_out/rf_launches.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/rf_ncu_launches.log 2>&1
