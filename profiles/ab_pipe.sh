#!/bin/bash
# software-pipelined long-row SELL sweeps (SMG_SELL_PIPE = 0 off, 4 / 6 = batch depth)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layouts.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_pipe.log 2>&1
echo "pytest(pipe default)=$?" >> gpurun_out/rc_pipe.txt
SMG_SELL_PIPE=6 timeout 900 python -m pytest tests/test_gpu_layouts.py -x -q > gpurun_out/pytest_pipe6.log 2>&1
echo "pytest(pipe6)=$?" >> gpurun_out/rc_pipe.txt
for w in C2 C4; do
  for p in 0 4 6; do
    SMG_SELL_PIPE=$p timeout 900 python bench.py --workload $w --steps 200 --warmup 5 --no-cpu-baseline \
      > gpurun_out/bench_${w}_pipe$p.json 2> gpurun_out/bench_${w}_pipe$p.err
    echo "$w pipe=$p rc=$?" >> gpurun_out/rc_pipe.txt
  done
done
