#!/bin/bash
# coarse solve: two PDL kernels (default) vs one fused kernel (SMG_COARSE_FUSED=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_coarse2.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_coarse2.txt
for w in C1 C3 C2; do
  for f in 0 1; do
    SMG_COARSE_FUSED=$f timeout 900 python bench.py --workload $w --steps 300 --warmup 10 --no-cpu-baseline \
      > gpurun_out/bench_${w}_cf$f.json 2> gpurun_out/bench_${w}_cf$f.err
    echo "$w fused=$f rc=$?" >> gpurun_out/rc_coarse2.txt
  done
done
