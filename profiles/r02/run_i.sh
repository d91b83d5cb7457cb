#!/bin/bash
# small-level tile sizing A/B on the current code (C2 and C3)
mkdir -p gpurun_out
for wl in C2 C3; do
for t in 4 8 16; do
  SMG_TILES_PER_SM=$t timeout 600 python bench.py --workload $wl --steps 300 --warmup 10 \
    > gpurun_out/ab_tiles_${wl}_$t.json 2> gpurun_out/ab_tiles_${wl}_$t.err
done
done
