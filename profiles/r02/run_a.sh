#!/bin/bash
# round-2 GPU session A: x-prefetch A/B (C2, C4), default bench, ncu of C2
mkdir -p gpurun_out
for wl in C2 C4; do
  for v in 0 1; do
    SMG_X_PREFETCH=$v timeout 900 python bench.py --workload $wl --steps 200 --warmup 10 \
      --skip-extras --device-assembly > gpurun_out/ab_xpf_${wl}_$v.json 2> gpurun_out/ab_xpf_${wl}_$v.err
  done
done
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "bench=$?" >> gpurun_out/rc.txt
timeout 1800 bash profiles/run_ncu.sh r02a >> gpurun_out/rc.txt 2>&1
