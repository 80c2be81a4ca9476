#!/bin/bash
# Round 2 final evidence on the final kernels: GPU suite (fast + full, parity report), smoke,
# C2 driver form (--steps 20) and 600 steps, C3/C4/C5, fixed N = 320, ncu launch list of the
# C2 command, ncu --set full of the one-slice scan and the tail, compute-sanitizer memcheck.
set -u
OUT=gpurun_out/final
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
export ARGUS_PARITY_REPORT=$OUT/parity_report.jsonl
rm -f $ARGUS_PARITY_REPORT
timeout 1200 python -m pytest tests -m "gpu and not full" -q -p no:cacheprovider > $OUT/pytest_fast.log 2>&1; echo "rc=$?" >> $OUT/pytest_fast.log
timeout 1500 python -m pytest tests -m full -q -p no:cacheprovider > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
unset ARGUS_PARITY_REPORT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_C2_s20_$rep.log 2>&1
  timeout 600 python bench.py --steps 600 --warmup 5 --no-cpu-baseline > $OUT/bench_C2_s600_$rep.log 2>&1
done
for C in C3 C4 C5; do timeout 600 python bench.py --config $C --steps 40 --warmup 5 --no-cpu-baseline > $OUT/bench_$C.log 2>&1; done
timeout 600 python bench.py --fixed-n 320 --steps 40 --warmup 5 --no-cpu-baseline --tensor-n 0 > $OUT/bench_N320.log 2>&1
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 200 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --tensor-n 0 > $OUT/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_tc -s 12 -c 1 \
   -o $OUT/prof_scan_N64 -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --tensor-n 0 \
   --e2e-steps 1 --fixed-n 64 > $OUT/ncu_scan_N64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 10 -c 1 \
   -o $OUT/prof_tail_N48 -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --pipeline 0 --tensor-n 0 \
   --e2e-steps 1 --fixed-n 48 > $OUT/ncu_tail_N48.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --target-processes all python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_parity.py tests/test_gpu_parity_exact.py tests/test_gpu_control.py tests/test_gpu_lifecycle.py \
  tests/test_gpu_nccl_path.py -m "gpu and not full" > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
tail -2 $OUT/pytest_fast.log $OUT/pytest_full.log $OUT/smoke.log $OUT/memcheck.log
