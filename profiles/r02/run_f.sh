#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/c5_patch_sweep.py > gpurun_out/c5_empty.jsonl 2> gpurun_out/c5_empty.err
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/t_fast.log 2>&1
echo "fast=$?" >> gpurun_out/rc.txt
SMG_LIB=paper_2402_12947_b200/lib/libsimplexmg_b200_checked.so timeout 900 python tools/sanitize_driver.py --mode default > gpurun_out/checked_empty.log 2>&1
echo "checked=$?" >> gpurun_out/rc.txt
timeout 900 python tools/sanitize_driver.py --mode default --stress 30 > gpurun_out/stress_empty.log 2>&1
echo "stress=$?" >> gpurun_out/rc.txt
