#!/bin/bash
# round-2 GPU session B: fine-level SELL variants (C2), patch-ring depth (C5 sweep)
mkdir -p gpurun_out
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 600 python bench.py --workload C2 --steps 300 --warmup 10 --skip-extras \
    > gpurun_out/ab_sell_$tag.json 2> gpurun_out/ab_sell_$tag.err
}
run base
run long8pipe6 SMG_SELL_MAX_ROW=0
run long8pipe4 SMG_SELL_MAX_ROW=0 SMG_SELL_PIPE=4
run long8plain SMG_SELL_MAX_ROW=0 SMG_SELL_PIPE=0
for st in 2 3 4 6; do
  SMG_PATCH_STAGES=$st timeout 600 python tools/c5_patch_sweep.py > gpurun_out/c5_stages_$st.jsonl 2> gpurun_out/c5_stages_$st.err
done
