#!/bin/bash
# GPU tests, then A/B of the LC/interior-sweep overlap (SMG_LC_SPLIT=0 disables it)
# on C1/C2/C3.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/rc.txt
for w in C2 C3 C1; do
  for split in 1 0; do
    SMG_LC_SPLIT=$split timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline \
      > gpurun_out/bench_${w}_split$split.json 2> gpurun_out/bench_${w}_split$split.err
    echo "$w split=$split rc=$?" >> gpurun_out/rc.txt
  done
done
