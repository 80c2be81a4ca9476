#!/bin/bash
# ncu --set full on the small kernels of one routing step (fixed N), one launch each.
set -u
OUT=gpurun_out
mkdir -p $OUT
ARGS="--steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fixed-n ${PN:-96}"
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"${PK:-k_mlp|k_merge_topk|k_assign|k_prep_queries}" -s ${PSKIP:-40} -c ${PCAP:-5} \
   -o $OUT/prof_small -f python bench.py $ARGS > $OUT/ncu_small.log 2>&1
echo "small rc=$?" >> $OUT/ncu_small.log
