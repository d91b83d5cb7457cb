#!/bin/bash
# C2 level 1 (SELL 8-deep, 1,029 windows): pipeline depth re-check with the carve-out in place; tile size for level 2
O=gpurun_out/ai
mkdir -p $O
for pp in 6 4 0; do
  SMG_SELL_PIPE=$pp timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --skip-extras > $O/bench_C2_pipe$pp.json 2> $O/bench_C2_pipe$pp.err
  echo "C2_pipe$pp=$?" >> $O/rc.txt
done
for ts in 3 6; do
  SMG_TILES_PER_SM=$ts timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --skip-extras > $O/bench_C2_tps$ts.json 2> $O/bench_C2_tps$ts.err
  echo "C2_tps$ts=$?" >> $O/rc.txt
done
