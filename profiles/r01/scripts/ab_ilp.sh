#!/bin/bash
# independent partial sums in the patch triangular solves: parity, trace, C2/C3 LC, C5 patches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_ilp.txt
python tools/trace_patch.py run c3s c2s c5 > gpurun_out/trace_patch4.json 2> gpurun_out/trace_patch4.err
for w in C2 C3; do
  timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/ilp_$w.json 2> gpurun_out/ilp_$w.err
  echo "$w rc=$?" >> gpurun_out/rc_ilp.txt
done
timeout 900 python bench.py --workload C5 --steps 50 --warmup 5 --no-cpu-baseline --c5-grids 63 > gpurun_out/ilp_C5.json 2> gpurun_out/ilp_C5.err
echo "C5 rc=$?" >> gpurun_out/rc_ilp.txt
