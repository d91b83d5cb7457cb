#!/bin/bash
# byte-ring streamed patch solves + own-dof prefetch: parity, trace, C2/C3 bench,
# C5 patches at ring capacities 2/3/4 longest chunks (SMG_PATCH_RING)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/rc.txt
python tools/trace_patch.py run c3s c2s c1s c5 > gpurun_out/trace_patch3.json 2> gpurun_out/trace_patch3.err
for w in C2 C3; do
  timeout 900 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline \
    > gpurun_out/ring_$w.json 2> gpurun_out/ring_$w.err
  echo "$w rc=$?" >> gpurun_out/rc.txt
done
for r in 2 3 4; do
  SMG_PATCH_RING=$r timeout 900 python bench.py --workload C5 --steps 100 --warmup 5 --no-cpu-baseline --c5-grids 63 \
    > gpurun_out/ring_C5_r$r.json 2> gpurun_out/ring_C5_r$r.err
  echo "C5 ring=$r rc=$?" >> gpurun_out/rc.txt
done
