#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layouts.py -q -x -k renumbered > gpurun_out/t_renum.log 2>&1
echo "trenum=$?" >> gpurun_out/rc.txt
for wl in C4 C2; do
for m in 0 1; do
  SMG_RENUMBER=$m timeout 900 python bench.py --workload $wl --steps 200 --warmup 10 --skip-extras \
    --device-assembly > gpurun_out/ab_cluster_${wl}_$m.json 2> gpurun_out/ab_cluster_${wl}_$m.err
done
done
