#!/bin/bash
# sym path (8-row chunks, column blocks, butterfly): trace, tests, C5 sweep; delta-coded SELL with relaxed register bounds
mkdir -p gpurun_out/o
timeout 600 python tools/trace_sym.py > gpurun_out/o/trace_sym.jsonl 2> gpurun_out/o/trace_sym.err
echo "trace=$?" > gpurun_out/o/rc.txt
timeout 900 python -m pytest tests/test_gpu_patch_sym.py tests/test_gpu_multiregion.py -q -x -m gpu > gpurun_out/o/pytest_sym.log 2>&1
echo "pytest_sym=$?" >> gpurun_out/o/rc.txt
timeout 600 python tools/c5_patch_sweep.py > gpurun_out/o/c5_sweep_sym1.jsonl 2> gpurun_out/o/c5_sweep_sym1.err
echo "sweep1=$?" >> gpurun_out/o/rc.txt
for kb in 100 132; do
  SMG_SYM_RING_KB=$kb timeout 300 python tools/c5_patch_sweep.py --case C5 > gpurun_out/o/c5_ring${kb}.jsonl 2>&1
done
SMG_LIB=paper_2402_12947_b200/lib/libsimplexmg_b200_d16relax.so timeout 900 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --skip-extras > gpurun_out/o/bench_C2_d16relax.json 2> gpurun_out/o/bench_C2_d16relax.err
echo "bench_relax=$?" >> gpurun_out/o/rc.txt
timeout 900 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --skip-extras > gpurun_out/o/bench_C2_d16.json 2> gpurun_out/o/bench_C2_d16.err
echo "bench_d16=$?" >> gpurun_out/o/rc.txt
