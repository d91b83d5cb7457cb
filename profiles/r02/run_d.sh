#!/bin/bash
# round-2 GPU session D: streamed patch solve after the chunk-cursor rewrite (8-row product
# build) and the 16-row variant
mkdir -p gpurun_out
timeout 600 python tools/c5_patch_sweep.py > gpurun_out/c5_cursor8.jsonl 2> gpurun_out/c5_cursor8.err
SMG_LIB=paper_2402_12947_b200/lib/libsimplexmg_b200_chunk16.so timeout 600 python tools/c5_patch_sweep.py \
  > gpurun_out/c5_cursor16.jsonl 2> gpurun_out/c5_cursor16.err
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c5 or vcycles or sandwich" > gpurun_out/t_patch.log 2>&1
echo "tpatch=$?" >> gpurun_out/rc.txt
