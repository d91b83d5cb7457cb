#!/bin/bash
# coarse solve as ONE kernel (last-CTA row reduction, PDL): GPU suite + benches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_coarse1.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_coarse1.txt
for w in C1 C3 C2 C4; do
  timeout 900 python bench.py --workload $w --steps 300 --warmup 10 --no-cpu-baseline \
    > gpurun_out/bench_${w}_coarse1.json 2> gpurun_out/bench_${w}_coarse1.err
  echo "$w rc=$?" >> gpurun_out/rc_coarse1.txt
done
