#!/bin/bash
# SELL (pipelined 8-deep) for smaller long-row operators: SMG_SELL_MIN_WIN_LONG
# 592 (default) / 200 / 60 on C2, C3, C4
mkdir -p gpurun_out
for w in C2 C3 C4; do
  for mw in 592 200 60; do
    SMG_SELL_MIN_WIN_LONG=$mw timeout 900 python bench.py --workload $w --steps 200 --warmup 5 --no-cpu-baseline \
      > gpurun_out/bench_${w}_mw$mw.json 2> gpurun_out/bench_${w}_mw$mw.err
    echo "$w minwin=$mw rc=$?" >> gpurun_out/rc_minwin.txt
  done
done
