#!/bin/bash
# streamed patch solve: is the single-patch latency copy-bound?  (L2 prefetch of
# the whole factor, ring depth) + coarse factor timing at C4 size
mkdir -p gpurun_out
for v in "" "SMG_PATCH_L2PF=1" "SMG_PATCH_STAGES=4" "SMG_PATCH_L2PF=1 SMG_PATCH_STAGES=4"; do
  echo "== $v" >> gpurun_out/c5_lat.jsonl
  env $v timeout 300 python tools/c5_patch_sweep.py --case "512 x1" >> gpurun_out/c5_lat.jsonl 2>&1
  env $v timeout 300 python tools/c5_patch_sweep.py --case "C5" >> gpurun_out/c5_lat.jsonl 2>&1
done
timeout 900 python tools/bench_coarse_factor.py > gpurun_out/coarse_factor.json 2> gpurun_out/coarse_factor.err
echo "coarse=$?" >> gpurun_out/rc.txt
