#!/bin/bash
# follow-mode corrections with a shared-memory carveout on the SELL sweeps
mkdir -p gpurun_out
for w in C3 C2; do
  for cfg in "1 -1" "1 50" "1 100" "0 -1" "0 50"; do
    set -- $cfg
    SMG_LC_FOLLOW=$1 SMG_SELL_CARVEOUT=$2 timeout 900 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline \
      > gpurun_out/bench_${w}_f$1_c$2.json 2> gpurun_out/bench_${w}_f$1_c$2.err
    echo "$w follow=$1 carve=$2 rc=$?" >> gpurun_out/rc_follow2.txt
  done
done
