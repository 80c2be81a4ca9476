#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/walk_bench > gpurun_out/walk_bench.txt 2>&1
echo rc=$? >> gpurun_out/walk_bench.txt
