#!/bin/bash
# sym path with full/empty mbarrier ring (4-row chunks): tests, C5 sweep, ring depth A/B, then the whole GPU suite
mkdir -p gpurun_out/p
timeout 600 python -m pytest tests/test_gpu_patch_sym.py tests/test_gpu_multiregion.py -q -x -m gpu > gpurun_out/p/pytest_sym.log 2>&1
echo "pytest_sym=$?" > gpurun_out/p/rc.txt
timeout 600 python tools/c5_patch_sweep.py > gpurun_out/p/c5_sweep_sym1.jsonl 2> gpurun_out/p/c5_sweep_sym1.err
echo "sweep1=$?" >> gpurun_out/p/rc.txt
for kb in 34 50 82 100; do
  SMG_SYM_RING_KB=$kb timeout 300 python tools/c5_patch_sweep.py --case C5 > gpurun_out/p/c5_ring${kb}.jsonl 2>&1
done
timeout 2400 python -m pytest tests -q -x -m gpu > gpurun_out/p/pytest_gpu.log 2>&1
echo "pytest=$?" >> gpurun_out/p/rc.txt
timeout 1200 python bench.py --workload C4 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/p/bench_C4.json 2> gpurun_out/p/bench_C4.err
echo "bench_C4=$?" >> gpurun_out/p/rc.txt
