#!/bin/bash
# staged tile kernel as two / three resident waves for C2 level 2
O=gpurun_out/ac
mkdir -p $O
for wv in 1 2 3; do
  SMG_STAGE_WAVES=$wv timeout 600 python tools/level_costs.py > $O/level_costs_C2_wv$wv.json 2>> $O/err.log
  SMG_STAGE_WAVES=$wv timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --skip-extras > $O/bench_C2_wv$wv.json 2> $O/bench_C2_wv$wv.err
  echo "C2_wv$wv=$?" >> $O/rc.txt
done
SMG_STAGE_WAVES=2 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "C2" > $O/pytest_full_wv2.log 2>&1
echo "pytest_full_wv2=$?" >> $O/rc.txt
