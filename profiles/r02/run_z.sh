#!/bin/bash
# Folded-chunk sym rings (SMG_SYM_FOLD=1): tests, C5 patch sweep fold x ring depth, C4 bench
O=gpurun_out/z
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_patch_sym.py tests/test_gpu_multiregion.py -q -x -m gpu > $O/pytest_sym.log 2>&1
echo "pytest_sym=$?" > $O/rc.txt
for ns in 2 3 4 6; do
  for cs in C5 512 384 256 192; do
    SMG_SYM_FOLD=1 SMG_SYM_STAGES=$ns timeout 300 python tools/c5_patch_sweep.py --case $cs >> $O/c5_fold1_st$ns.jsonl 2>> $O/err.log
  done
done
for cs in C5 512 384 256 192; do
  SMG_SYM_FOLD=0 timeout 300 python tools/c5_patch_sweep.py --case $cs >> $O/c5_fold0.jsonl 2>> $O/err.log
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -q -x -m gpu > $O/pytest_par.log 2>&1
echo "pytest_par=$?" >> $O/rc.txt
for fo in 0 1; do
  SMG_SYM_FOLD=$fo timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4_fold$fo.json 2> $O/bench_C4_fold$fo.err
  echo "C4_fold$fo=$?" >> $O/rc.txt
done
