#!/bin/bash
mkdir -p gpurun_out
python -m paper_2511_06724_b200.build > gpurun_out/build6.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not full" -q -x > gpurun_out/rc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/rc_smoke.log
for rep in 1 2; do timeout 600 python bench.py > gpurun_out/rc_bench_$rep.log 2>&1; done
timeout 300 python bench.py --no-cpu-baseline --fixed-n 48 --steps 2000 > gpurun_out/rc_n48.log 2>&1
