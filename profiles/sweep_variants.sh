#!/bin/bash
# HISTORICAL: the SMG_SPMV_VARIANT kernels were removed after these A/Bs.
# A/B the SpMV kernel variants (SMG_SPMV_VARIANT) and PDL (SMG_PDL) on the C2 bench.
mkdir -p gpurun_out
for cfg in "1 1" "3 1" "4 1" "2 1" "1 0"; do
  set -- $cfg
  SMG_SPMV_VARIANT=$1 SMG_PDL=$2 timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline \
    > gpurun_out/bench_v$1_pdl$2.json 2> gpurun_out/bench_v$1_pdl$2.err
done
