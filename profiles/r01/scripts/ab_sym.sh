#!/bin/bash
# symmetric tiled coarse solve: GPU parity, C2/C3/C1 bench, then C4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_sym.txt
for w in C2 C3 C1; do
  timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/sym_$w.json 2> gpurun_out/sym_$w.err
  echo "$w rc=$?" >> gpurun_out/rc_sym.txt
done
timeout 1800 python bench.py --workload C4 --steps 100 --warmup 5 > gpurun_out/sym_C4.json 2> gpurun_out/sym_C4.err
echo "C4 rc=$?" >> gpurun_out/rc_sym.txt
