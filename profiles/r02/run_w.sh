#!/bin/bash
# (1) sym rings: L2 prefetch distance A/B; (2) warp-specialised tile kernel (SMG_TILE_WS=1): bitwise tests, C2/C3/C4 A/B
O=gpurun_out/w
mkdir -p $O
for pf in 0 2 4 8 16; do
  for cs in C5 512 256; do
    SMG_SYM_L2PF=$pf timeout 300 python tools/c5_patch_sweep.py --case $cs >> $O/c5_l2pf$pf.jsonl 2>> $O/err.log
  done
done
timeout 600 python -m pytest tests/test_gpu_patch_sym.py -q -x -m gpu > $O/pytest_sym.log 2>&1
echo "pytest_sym=$?" > $O/rc.txt
SMG_TILE_WS=1 timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layouts.py tests/test_gpu_properties.py tests/test_gpu_multiregion.py -q -x -m gpu > $O/pytest_ws.log 2>&1
echo "pytest_ws=$?" >> $O/rc.txt
SMG_TILE_WS=1 timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu > $O/pytest_ws_full.log 2>&1
echo "pytest_ws_full=$?" >> $O/rc.txt
for ws in 0 1; do
  SMG_TILE_WS=$ws timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_C2_ws$ws.json 2> $O/bench_C2_ws$ws.err
  echo "C2_ws$ws=$?" >> $O/rc.txt
  SMG_TILE_WS=$ws timeout 900 python bench.py --workload C3 --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_C3_ws$ws.json 2> $O/bench_C3_ws$ws.err
  echo "C3_ws$ws=$?" >> $O/rc.txt
done
for ws in 0 1; do
  SMG_TILE_WS=$ws timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C4_ws$ws.json 2> $O/bench_C4_ws$ws.err
  echo "C4_ws$ws=$?" >> $O/rc.txt
done
