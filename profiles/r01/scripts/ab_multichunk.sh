#!/bin/bash
# multi-chunk tiles for long-row operators (SMG_MC_MIN_ROW=0 disables):
# GPU parity, then A/B on C2, C3, C5 and C4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_mc.txt
for mc in 24 0; do
  for w in C2 C3; do
    SMG_MC_MIN_ROW=$mc timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/mc${mc}_$w.json 2> gpurun_out/mc${mc}_$w.err
    echo "$w mc=$mc rc=$?" >> gpurun_out/rc_mc.txt
  done
  SMG_MC_MIN_ROW=$mc timeout 900 python bench.py --workload C5 --steps 100 --warmup 5 --no-cpu-baseline --c5-grids 63,126 > gpurun_out/mc${mc}_C5.json 2> gpurun_out/mc${mc}_C5.err
  echo "C5 mc=$mc rc=$?" >> gpurun_out/rc_mc.txt
done
SMG_MC_MIN_ROW=24 timeout 1800 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/mc24_C4.json 2> gpurun_out/mc24_C4.err
echo "C4 rc=$?" >> gpurun_out/rc_mc.txt
