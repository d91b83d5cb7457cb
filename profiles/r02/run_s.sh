#!/bin/bash
# sym path v6 (two blocks per warp pass) + persisting-L2 window for the gathered vector (SMG_L2_PERSIST_MB) A/B on C2 and C4
O=gpurun_out/s
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_patch_sym.py tests/test_gpu_multiregion.py -q -x -m gpu > $O/pytest_sym.log 2>&1
echo "pytest_sym=$?" > $O/rc.txt
timeout 600 python tools/c5_patch_sweep.py > $O/c5_sweep.jsonl 2> $O/c5_sweep.err
echo "sweep=$?" >> $O/rc.txt
timeout 600 python tools/trace_sym.py > $O/trace_sym.jsonl 2> $O/trace_sym.err
for mb in 0 24 48 90; do
  SMG_L2_PERSIST_MB=$mb timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --skip-extras > $O/bench_C2_persist$mb.json 2> $O/bench_C2_persist$mb.err
  echo "C2_persist$mb=$?" >> $O/rc.txt
done
for mb in 0 64 90; do
  SMG_L2_PERSIST_MB=$mb timeout 1500 python bench.py --workload C4 --steps 100 --warmup 5 --no-cpu-baseline --skip-extras > $O/bench_C4_persist$mb.json 2> $O/bench_C4_persist$mb.err
  echo "C4_persist$mb=$?" >> $O/rc.txt
done
