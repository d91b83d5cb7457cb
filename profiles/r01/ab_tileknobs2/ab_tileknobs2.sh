#!/bin/bash
# tile-kernel knobs re-measured on the final C2 (levels 2-3 run the tiles)
mkdir -p gpurun_out
for cfg in "base" "SMG_TILES_PER_SM=2" "SMG_TILES_PER_SM=8" "SMG_MC_CHUNKS=2" "SMG_PF_WAVES=2"; do
  if [ "$cfg" = "base" ]; then e=""; else e="$cfg"; fi
  env $e timeout 600 python bench.py --workload C2 --steps 500 --warmup 10 --no-cpu-baseline \
    > gpurun_out/bench_C2_tk_${cfg//=/_}.json 2> gpurun_out/bench_C2_tk_${cfg//=/_}.err
  echo "$cfg rc=$?" >> gpurun_out/rc_tk2.txt
done
