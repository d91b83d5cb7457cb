#!/bin/bash
# parallel panel GEMV in the patch solves: parity, phase trace, C2/C3/C5 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/rc.txt
python tools/trace_patch.py run c3s c2s c1s > gpurun_out/trace_patch2.json 2> gpurun_out/trace_patch2.err
for w in C2 C3 C5; do
  timeout 900 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline --c5-grids 63 \
    > gpurun_out/gemv_$w.json 2> gpurun_out/gemv_$w.err
  echo "$w rc=$?" >> gpurun_out/rc.txt
done
