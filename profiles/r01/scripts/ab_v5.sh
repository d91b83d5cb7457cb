#!/bin/bash
# HISTORICAL: the SMG_SPMV_VARIANT kernels were removed after these A/Bs.
mkdir -p gpurun_out
SMG_SPMV_VARIANT=12 timeout 900 python -m pytest tests -x -q -m gpu -k "sparse or sweep or vcycle" > gpurun_out/pytest_v12.log 2>&1
echo "v12 pytest rc=$?" >> gpurun_out/rc.txt
for v in 10 12; do
  SMG_SPMV_VARIANT=$v timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/bench_ab_v$v.json 2> gpurun_out/bench_ab_v$v.err
done
