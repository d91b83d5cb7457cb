#!/bin/bash
# register-resident symmetric-inverse apply (SMG_SYM_REG=1): tests, C5 patch sweep A/B, C4 / C2 bench
O=gpurun_out/ad
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_patch_sym.py tests/test_gpu_multiregion.py -q -x -m gpu > $O/pytest_sym.log 2>&1
echo "pytest_sym=$?" > $O/rc.txt
for rg in 1 0; do
  timeout 600 env SMG_SYM_REG=$rg python tools/c5_patch_sweep.py > $O/c5_reg$rg.jsonl 2>> $O/err.log
done
for ns in 3 4; do
  for cs in C5 512 256; do
    SMG_SYM_STAGES=$ns timeout 300 python tools/c5_patch_sweep.py --case $cs >> $O/c5_reg1_st$ns.jsonl 2>> $O/err.log
  done
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -q -x -m gpu > $O/pytest_par.log 2>&1
echo "pytest_par=$?" >> $O/rc.txt
for rg in 0 1; do
  SMG_SYM_REG=$rg timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4_reg$rg.json 2> $O/bench_C4_reg$rg.err
  echo "C4_reg$rg=$?" >> $O/rc.txt
done
timeout 900 python bench.py --workload C5 --steps 100 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
echo "bench_C5=$?" >> $O/rc.txt
