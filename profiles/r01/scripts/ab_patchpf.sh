#!/bin/bash
# C5 patch solves: L2 prefetch window of streamed factor chunks (SMG_PATCH_PF_CHUNKS)
mkdir -p gpurun_out
for pf in 0 2 3 6; do
  SMG_PATCH_PF_CHUNKS=$pf timeout 900 python bench.py --workload C5 --steps 50 --warmup 5 --no-cpu-baseline --c5-grids 63 > gpurun_out/ppf_$pf.json 2> gpurun_out/ppf_$pf.err
  echo "pf=$pf rc=$?" >> gpurun_out/rc_ppf.txt
done
timeout 600 python -m pytest tests -x -q -m gpu -k "c5 or sandwich or local" > gpurun_out/pytest_ppf.log 2>&1
echo "pytest=$?" >> gpurun_out/rc_ppf.txt
