#!/bin/bash
# multi-chunk for streamed long-row operators with fewer chunks per tile
mkdir -p gpurun_out
for ch in 2 3; do
  SMG_MC_MAX_STREAM_ROW=0 SMG_MC_CHUNKS=$ch timeout 600 python bench.py --workload C2 --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/mc3_C2_ch$ch.json 2> gpurun_out/mc3_C2_ch$ch.err
  echo "C2 ch=$ch rc=$?" >> gpurun_out/rc_mc3.txt
done
for ch in 2 3; do
  SMG_MC_MAX_STREAM_ROW=0 SMG_MC_CHUNKS=$ch timeout 1800 python bench.py --workload C4 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/mc3_C4_ch$ch.json 2> gpurun_out/mc3_C4_ch$ch.err
  echo "C4 ch=$ch rc=$?" >> gpurun_out/rc_mc3.txt
done
