#!/bin/bash
# sym rings: per-phase cycle trace (thread 0) and the refill fence A/B
O=gpurun_out/ab
mkdir -p $O
tools/micro/fp64_rate > $O/fp64_rate.jsonl 2>&1
timeout 600 python tools/trace_sym.py > $O/trace_sym.jsonl 2> $O/trace_sym.err
echo "trace=$?" > $O/rc.txt
SMG_SYM_NOFENCE=1 timeout 600 python tools/trace_sym.py > $O/trace_sym_nofence.jsonl 2>> $O/trace_sym.err
for nf in 0 1; do
  for cs in C5 512 256; do
    SMG_SYM_NOFENCE=$nf timeout 300 python tools/c5_patch_sweep.py --case $cs >> $O/c5_nofence$nf.jsonl 2>> $O/err.log
  done
done
SMG_SYM_NOFENCE=1 timeout 900 python -m pytest tests/test_gpu_patch_sym.py -q -x -m gpu > $O/pytest_sym_nofence.log 2>&1
echo "pytest_nofence=$?" >> $O/rc.txt
