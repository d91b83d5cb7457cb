#!/bin/bash
# multi-chunk rule v2 (not for HBM-streamed operators averaging >= 36 nnz/row)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_mc2.txt
for w in C2 C3 C1; do
  timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/mc2_$w.json 2> gpurun_out/mc2_$w.err
  echo "$w rc=$?" >> gpurun_out/rc_mc2.txt
done
timeout 900 python bench.py --workload C5 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/mc2_C5.json 2> gpurun_out/mc2_C5.err
echo "C5 rc=$?" >> gpurun_out/rc_mc2.txt
timeout 1800 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/mc2_C4.json 2> gpurun_out/mc2_C4.err
echo "C4 rc=$?" >> gpurun_out/rc_mc2.txt
