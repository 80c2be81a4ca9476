#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/mma_bench > gpurun_out/mma_bench.txt 2>&1
echo rc=$? >> gpurun_out/mma_bench.txt
