#!/bin/bash
# sym rings: L2 prefetch distance A/B (SMG_SYM_L2PF rounds of eight chunks ahead)
O=gpurun_out/v
mkdir -p $O
for pf in 0 2 4 8 16; do
  for cs in C5 512 256; do
    SMG_SYM_L2PF=$pf timeout 300 python tools/c5_patch_sweep.py --case $cs >> $O/c5_l2pf$pf.jsonl 2>> $O/err.log
  done
done
timeout 600 python -m pytest tests/test_gpu_patch_sym.py -q -x -m gpu > $O/pytest_sym.log 2>&1
echo "pytest_sym=$?" > $O/rc.txt
