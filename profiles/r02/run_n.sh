#!/bin/bash
# sym path phase trace + renumber fix check + delta layout tests
mkdir -p gpurun_out/n
timeout 600 python tools/trace_sym.py > gpurun_out/n/trace_sym.jsonl 2> gpurun_out/n/trace_sym.err
echo "trace=$?" > gpurun_out/n/rc.txt
timeout 900 python -m pytest tests/test_gpu_patch_sym.py -q -x -m gpu > gpurun_out/n/pytest_sym.log 2>&1
echo "pytest_sym=$?" >> gpurun_out/n/rc.txt
timeout 1800 python -m pytest tests/test_gpu_layouts.py -q -x -m gpu > gpurun_out/n/pytest_layouts.log 2>&1
echo "pytest_layouts=$?" >> gpurun_out/n/rc.txt
timeout 900 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/n/bench_C2_delta.json 2> gpurun_out/n/bench_C2_delta.err
echo "bench_delta=$?" >> gpurun_out/n/rc.txt
SMG_SELL_DELTA=0 timeout 900 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/n/bench_C2_nodelta.json 2> gpurun_out/n/bench_C2_nodelta.err
echo "bench_nodelta=$?" >> gpurun_out/n/rc.txt
