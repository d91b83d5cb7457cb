#!/bin/bash
# whole-L^{-1} GEMVs for 65..128-dof regions (C2's 101-dof patches)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_linv128.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_linv128.txt
for w in C2 C3 C5; do
  timeout 900 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline \
    > gpurun_out/bench_${w}_linv128.json 2> gpurun_out/bench_${w}_linv128.err
  echo "$w rc=$?" >> gpurun_out/rc_linv128.txt
done
