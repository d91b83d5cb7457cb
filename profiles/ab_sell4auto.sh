#!/bin/bash
# SELL-8x4 (4 batches) only for operators with >= 200 nonzeros per row (C4 level 2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layouts.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_sell4auto.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_sell4auto.txt
for w in C4 C2 C3; do
  for m in 2 0; do
    SMG_SELL4=$m timeout 900 python bench.py --workload $w --steps 200 --warmup 5 --no-cpu-baseline \
      > gpurun_out/bench_${w}_s4auto$m.json 2> gpurun_out/bench_${w}_s4auto$m.err
    echo "$w sell4=$m rc=$?" >> gpurun_out/rc_sell4auto.txt
  done
done
