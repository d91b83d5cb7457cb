#!/bin/bash
# round-2 GPU session C: GPU tests (not slow), SELL variants A/B, ncu of the streamed patch solve
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/t_fast.log 2>&1
echo "fast=$?" >> gpurun_out/rc.txt
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 600 python bench.py --workload C2 --steps 300 --warmup 10 --skip-extras \
    > gpurun_out/ab_sell_$tag.json 2> gpurun_out/ab_sell_$tag.err
}
run base
run long8pipe6 SMG_SELL_MAX_ROW=0
run long8pipe4 SMG_SELL_MAX_ROW=0 SMG_SELL_PIPE=4
run long8plain SMG_SELL_MAX_ROW=0 SMG_SELL_PIPE=0
timeout 300 python tools/c5_patch_sweep.py --case "512 x1" --reps 3 > gpurun_out/c5_512x1_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:patch_kernel -c 2 \
  -o gpurun_out/prof_patch512_r02c python tools/c5_patch_sweep.py --case "512 x1" --reps 1 \
  > gpurun_out/ncu_patch512.log 2>&1
echo "ncu512=$?" >> gpurun_out/rc.txt
