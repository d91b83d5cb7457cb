#!/bin/bash
# staged tile kernel: which operators (SMG_STAGE_MAX_CAP) -- C2 level costs and bench, C3 bench; carve-out on (default)
O=gpurun_out/aa
mkdir -p $O
for mc in 1 3500 4096 9216; do
  SMG_STAGE_MAX_CAP=$mc timeout 600 python tools/level_costs.py > $O/level_costs_C2_mc$mc.json 2>> $O/err.log
  SMG_STAGE_MAX_CAP=$mc timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --skip-extras > $O/bench_C2_mc$mc.json 2> $O/bench_C2_mc$mc.err
  echo "C2_mc$mc=$?" >> $O/rc.txt
  SMG_STAGE_MAX_CAP=$mc timeout 900 python bench.py --workload C3 --steps 300 --warmup 10 --no-cpu-baseline --skip-extras > $O/bench_C3_mc$mc.json 2> $O/bench_C3_mc$mc.err
  SMG_STAGE_MAX_CAP=$mc timeout 900 python bench.py --workload C1 --steps 300 --warmup 10 --no-cpu-baseline --skip-extras > $O/bench_C1_mc$mc.json 2> $O/bench_C1_mc$mc.err
done
