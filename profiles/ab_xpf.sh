#!/bin/bash
# A/B: SMG_X_PREFETCH (x pulled into L2 after the dependency wait) on C2, C4, C5
mkdir -p gpurun_out
for wl in C2 C4; do
  for v in 0 1; do
    SMG_X_PREFETCH=$v timeout 900 python bench.py --workload $wl --steps 200 --warmup 10 \
      --skip-extras --device-assembly > gpurun_out/ab_xpf_${wl}_$v.json 2> gpurun_out/ab_xpf_${wl}_$v.err
  done
done
for v in 0 1; do
  SMG_X_PREFETCH=$v timeout 900 python bench.py --workload C5 --steps 100 \
    > gpurun_out/ab_xpf_C5_$v.json 2> gpurun_out/ab_xpf_C5_$v.err
done
