#!/bin/bash
# sym path v4 (8-row chunks, CTA barrier, refill prepared before the barrier, two column chains): tests, trace, C5 sweep, ncu of the C5 patch kernel;
# SELL-d16 vs int32 columns: ncu of the C2 sweeps under SMG_SELL_DELTA=1
mkdir -p gpurun_out/q
timeout 600 python -m pytest tests/test_gpu_patch_sym.py tests/test_gpu_multiregion.py -q -x -m gpu > gpurun_out/q/pytest_sym.log 2>&1
echo "pytest_sym=$?" > gpurun_out/q/rc.txt
timeout 600 python tools/trace_sym.py > gpurun_out/q/trace_sym.jsonl 2> gpurun_out/q/trace_sym.err
timeout 600 python tools/c5_patch_sweep.py > gpurun_out/q/c5_sweep_sym1.jsonl 2> gpurun_out/q/c5_sweep_sym1.err
echo "sweep1=$?" >> gpurun_out/q/rc.txt
CMD="python tools/c5_patch_sweep.py --case C5 --reps 3"
$CMD > gpurun_out/q/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:patch_kernel -s 3 -c 1 -o gpurun_out/q/prof_patchC5_r02q $CMD > gpurun_out/q/ncu_c5.log 2>&1
echo "ncu_c5=$?" >> gpurun_out/q/rc.txt
export SMG_SELL_DELTA=1
if timeout 900 python tools/profile_driver.py > gpurun_out/q/plain_d16.log 2>&1; then
  timeout 1200 ncu --nvtx --nvtx-include "sweeps/" -k regex:"sell_kernel" --launch-count 2 --set full --clock-control none --import-source on \
     -o gpurun_out/q/prof_sweeps_d16_r02q python tools/profile_driver.py > gpurun_out/q/ncu_d16.log 2>&1
  echo "ncu_d16=$?" >> gpurun_out/q/rc.txt
fi
unset SMG_SELL_DELTA
timeout 1200 ncu --nvtx --nvtx-include "sweeps/" -k regex:"sell_kernel" --launch-count 2 --set full --clock-control none --import-source on \
     -o gpurun_out/q/prof_sweeps_i32_r02q python tools/profile_driver.py > gpurun_out/q/ncu_i32.log 2>&1
echo "ncu_i32=$?" >> gpurun_out/q/rc.txt
