#!/bin/bash
# sym path v7b (grouped loads): tests and C5 sweep
O=gpurun_out/u
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_patch_sym.py tests/test_gpu_multiregion.py -q -x -m gpu > $O/pytest_sym.log 2>&1
echo "pytest_sym=$?" > $O/rc.txt
timeout 600 python tools/c5_patch_sweep.py > $O/c5_sweep.jsonl 2> $O/c5_sweep.err
echo "sweep=$?" >> $O/rc.txt
