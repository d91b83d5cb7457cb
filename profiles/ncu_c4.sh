#!/bin/bash
# ncu --set full of C4's fine-level sweep (first sweep in the driver's "sweeps" range)
OUT=gpurun_out; mkdir -p $OUT
CMD="python tools/profile_driver.py --workload C4"
if ! timeout 900 $CMD > $OUT/plain_c4.log 2>&1; then echo "plain run failed"; exit 1; fi
timeout 1500 ncu --nvtx --nvtx-include "sweeps/" -k regex:"sell_kernel" -c 1 --set full --clock-control none --import-source on \
    -o $OUT/prof_sweeps_c4 $CMD > $OUT/ncu_sweeps_c4.log 2>&1
echo "sweeps: $?"
