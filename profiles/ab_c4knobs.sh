#!/bin/bash
# C4 fine-level SELL loop depth: 8-deep (default for long rows), 16-deep,
# and 4-deep with 8 CTAs/SM (SMG_SELL_MAX_ROW=30 classes 26.5 nnz/row as short)
mkdir -p gpurun_out
for cfg in "def" "u16" "short30"; do
  case $cfg in
    def) env="" ;;
    u16) env="SMG_SELL_LONG_UNROLL=16" ;;
    short30) env="SMG_SELL_MAX_ROW=30" ;;
  esac
  env $env timeout 900 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline \
    > gpurun_out/bench_C4_$cfg.json 2> gpurun_out/bench_C4_$cfg.err
  echo "C4 $cfg rc=$?" >> gpurun_out/rc_c4knobs.txt
done
