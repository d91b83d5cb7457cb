#!/bin/bash
# ncu --set full of C4's level-2 ChebNext step (third launch of the 'sweeps' range): why 0.49 of HBM in every layout
O=gpurun_out/ag
mkdir -p $O
CMD="python tools/profile_driver.py --workload C4"
if timeout 1500 $CMD > $O/plain_C4.log 2>&1; then
  timeout 1800 ncu --nvtx --nvtx-include "sweeps/" -k regex:"csr_tile_kernel|sell_kernel|csr_stage_kernel" --launch-skip 1 --launch-count 2 --set full --clock-control none --import-source on -o $O/prof_sweep12_C4_r02g $CMD > $O/ncu_sweep12_C4.log 2>&1
  echo "ncu_C4_l12=$?" >> $O/rc.txt
fi
