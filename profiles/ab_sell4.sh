#!/bin/bash
# SELL-8x4 (4 lanes per row) for long-row operators the SELL-32 rule leaves to
# the tiles: layout tests, then A/B (SMG_SELL4=0 keeps the tiles) on C2/C3/C1/C4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layouts.py -x -q > gpurun_out/pytest_layouts_sell4.log 2>&1
echo "pytest_layouts=$?" >> gpurun_out/rc_sell4.txt
for w in C2 C3 C1 C4; do
  for cfg in "1 2" "1 4" "0 2"; do
    set -- $cfg
    if [ "$w" = "C4" ] && [ "$2" = "4" ]; then continue; fi
    SMG_SELL4=$1 SMG_SELL4_UNROLL=$2 timeout 900 python bench.py --workload $w --steps 300 --warmup 10 --no-cpu-baseline \
      > gpurun_out/bench_${w}_s4_$1_$2.json 2> gpurun_out/bench_${w}_s4_$1_$2.err
    echo "$w sell4=$1 unroll=$2 rc=$?" >> gpurun_out/rc_sell4.txt
  done
done
