#!/bin/bash
# Round-end evidence: all GPU tests, smoke, one bench line per config, ncu of the scans.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2511_06724_b200.build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not full" -q -x > $OUT/pytest_fast.log 2>&1; echo "rc=$?" >> $OUT/pytest_fast.log
timeout 1200 python -m pytest tests -m full -q > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_C2.log 2>&1
for C in C5 C3 C4; do timeout 600 python bench.py --config $C --steps 40 --warmup 5 > $OUT/bench_$C.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 200 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_launches.log 2>&1
for spec in "C2:64:k_scan_tc" "C2:256:k_scan_pair" "C5:4096:k_scan_pair" "C4:8192:k_scan_pair" "C3:256:k_scan_pair"; do
  C=$(echo $spec | cut -d: -f1); N=$(echo $spec | cut -d: -f2); K=$(echo $spec | cut -d: -f3)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 6 -c 1 \
     -o $OUT/prof_${C}_N$N -f python bench.py --config $C --steps 4 --warmup 3 --no-cpu-baseline \
     --e2e-steps 1 --fixed-n $N > $OUT/ncu_${C}_N$N.log 2>&1
done
