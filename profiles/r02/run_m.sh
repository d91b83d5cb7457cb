#!/bin/bash
# symmetric-inverse patch path: new tests first, C5 sweep under both settings, then the whole suite
mkdir -p gpurun_out/m
timeout 900 python -m pytest tests/test_gpu_patch_sym.py tests/test_gpu_multiregion.py -q -x -m gpu > gpurun_out/m/pytest_sym.log 2>&1
echo "pytest_sym=$?" > gpurun_out/m/rc.txt
timeout 600 python tools/c5_patch_sweep.py > gpurun_out/m/c5_sweep_sym1.jsonl 2> gpurun_out/m/c5_sweep_sym1.err
echo "sweep1=$?" >> gpurun_out/m/rc.txt
SMG_PATCH_SYM=0 timeout 600 python tools/c5_patch_sweep.py > gpurun_out/m/c5_sweep_sym0.jsonl 2> gpurun_out/m/c5_sweep_sym0.err
echo "sweep0=$?" >> gpurun_out/m/rc.txt
for kb in 32 96; do
  SMG_SYM_RING_KB=$kb timeout 300 python tools/c5_patch_sweep.py --case C5 > gpurun_out/m/c5_ring${kb}.jsonl 2>&1
done
for st in 1024 4096; do
  SMG_SYM_STAGE=$st timeout 300 python tools/c5_patch_sweep.py --case C5 > gpurun_out/m/c5_stage${st}.jsonl 2>&1
done
timeout 2400 python -m pytest tests -q -x -m gpu > gpurun_out/m/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/m/rc.txt
timeout 1200 python bench.py --workload C4 --steps 200 --warmup 10 > gpurun_out/m/bench_C4.json 2> gpurun_out/m/bench_C4.err
echo "bench_C4=$?" >> gpurun_out/m/rc.txt
timeout 900 python bench.py --workload C5 --steps 100 > gpurun_out/m/bench_C5.json 2> gpurun_out/m/bench_C5.err
echo "bench_C5=$?" >> gpurun_out/m/rc.txt
