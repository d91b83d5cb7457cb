#!/bin/bash
# Per-config bench records (C1, C3, C4, C5) with the CPU oracle beside them.
# Usage: bash profiles/configs_bench.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
for w in C1 C3 C4 C5; do
  timeout 1200 python bench.py --workload $w --steps 300 --warmup 10 \
    > gpurun_out/bench_${w}_$TAG.json 2> gpurun_out/bench_${w}_$TAG.err
  echo "$w rc=$?" >> gpurun_out/rc_configs_$TAG.txt
done
