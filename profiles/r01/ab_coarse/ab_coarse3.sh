#!/bin/bash
# coarse solve: block-row-parallel reduction (default now); tiles evict-first
# (default) vs normal L2 priority (SMG_COARSE_KEEP=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_coarse3.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_coarse3.txt
for w in C2 C1 C3; do
  for k in 0 1; do
    SMG_COARSE_KEEP=$k timeout 900 python bench.py --workload $w --steps 300 --warmup 10 --no-cpu-baseline \
      > gpurun_out/bench_${w}_ck$k.json 2> gpurun_out/bench_${w}_ck$k.err
    echo "$w keep=$k rc=$?" >> gpurun_out/rc_coarse3.txt
  done
done
