#!/bin/bash
# (1) L1/shared carve-out per launch x staged tile kernel: C2 bench + level costs; (2) sym ring depth sweep
O=gpurun_out/y
mkdir -p $O
for st in 0 1; do for cv in 0 1 2; do
  SMG_TILE_STAGE=$st SMG_CARVEOUT=$cv timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --skip-extras > $O/bench_C2_st${st}_cv$cv.json 2> $O/bench_C2_st${st}_cv$cv.err
  echo "C2_st${st}_cv$cv=$?" >> $O/rc.txt
  SMG_TILE_STAGE=$st SMG_CARVEOUT=$cv timeout 600 python tools/level_costs.py > $O/level_costs_C2_st${st}_cv$cv.json 2>> $O/err.log
done; done
for st in 0 1; do for cv in 0 1; do
  SMG_TILE_STAGE=$st SMG_CARVEOUT=$cv timeout 900 python bench.py --workload C3 --steps 300 --warmup 10 --no-cpu-baseline --skip-extras > $O/bench_C3_st${st}_cv$cv.json 2> $O/bench_C3_st${st}_cv$cv.err
done; done
for ns in 2 3 4; do
  for cs in C5 512 256; do
    SMG_SYM_STAGES=$ns timeout 300 python tools/c5_patch_sweep.py --case $cs >> $O/c5_stages$ns.jsonl 2>> $O/err.log
  done
done
