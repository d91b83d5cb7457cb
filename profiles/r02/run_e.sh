#!/bin/bash
mkdir -p gpurun_out
bash profiles/r02/checked_run.sh
SMG_PATCH_LPT=0 timeout 300 python tools/c5_patch_sweep.py --case C5 > gpurun_out/c5_lpt0.jsonl 2>&1
timeout 300 python tools/c5_patch_sweep.py --case C5 > gpurun_out/c5_lpt1.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:patch_kernel -c 1 \
  -o gpurun_out/prof_patchC5_r02e python tools/c5_patch_sweep.py --case C5 --reps 1 \
  > gpurun_out/ncu_patchC5.log 2>&1
echo "ncuC5=$?" >> gpurun_out/rc.txt
