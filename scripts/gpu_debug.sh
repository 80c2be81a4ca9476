#!/bin/bash
# Debug a failing path: error site with ARGUS_DEBUG, then compute-sanitizer memcheck on the smoke case.
mkdir -p gpurun_out
ARGUS_DEBUG=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/debug_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/debug_smoke.log
ARGUS_DEBUG=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/memcheck.log
