#!/bin/bash
# Round 2 evidence on the current code: all GPU tests (fast + full size), smoke, C2 with
# the driver's --steps 20 against --steps 600, C3/C4/C5 lines, ncu launch list of the C2
# bench and --set full captures of the tail.
set -u
OUT=gpurun_out
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
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 200 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --tensor-n 0 > $OUT/ncu_launches.log 2>&1
for N in 48 320; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 10 -c 1 \
   -o $OUT/prof_tail_N$N -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --pipeline 0 --tensor-n 0 \
   --e2e-steps 1 --fixed-n $N > $OUT/ncu_tail_N$N.log 2>&1
done
