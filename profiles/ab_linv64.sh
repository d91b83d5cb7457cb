#!/bin/bash
# whole-L^{-1} GEMVs for 33..64-dof regions: GPU suite, then C3/C1/C2/C4 benches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_linv64.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_linv64.txt
for w in C3 C1 C2; do
  timeout 900 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline \
    > gpurun_out/bench_${w}_linv64.json 2> gpurun_out/bench_${w}_linv64.err
  echo "$w rc=$?" >> gpurun_out/rc_linv64.txt
done
