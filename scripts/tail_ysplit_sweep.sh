mkdir -p gpurun_out
python -m paper_2511_06724_b200.build > gpurun_out/build3.log 2>&1
for rep in 1 2; do for y in 1 2 4; do
  ARGUS_TAIL_YSPLIT=$y timeout 300 python bench.py --no-cpu-baseline > gpurun_out/sw_y${y}_$rep.log 2>&1
done; done
