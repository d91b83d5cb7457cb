#!/bin/bash
# locality renumbering: bitwise test, then A/B on C2 and C4 (level masks)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layouts.py -q -x -k renumbered > gpurun_out/t_renum.log 2>&1
echo "trenum=$?" >> gpurun_out/rc.txt
for wl in C2 C4; do
for m in 0 1 3; do
  SMG_RENUMBER=$m timeout 900 python bench.py --workload $wl --steps 200 --warmup 10 --skip-extras \
    --device-assembly > gpurun_out/ab_renum_${wl}_$m.json 2> gpurun_out/ab_renum_${wl}_$m.err
done
done
